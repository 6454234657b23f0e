// asx_large.cuh — chirp-z α-DFT for signals whose cyclic FFT size P exceeds
// one CTA (BASELINE config 2: N = 2^22, α = 1/16, P = 2^23), as a four-step
// FFT P = P1 x P2 through an HBM/L2 workspace.
//
// Index maps (n = P2*n1 + n2, k = k1 + P1*k2 for the forward transform; the
// inverse reuses the transposed map k = k1 + P1*k2 -> n = c + P2*d):
//   KA  k_large_cols<FWD>: per tile of 8 columns n2, FFT_P1 over n1 of
//       y[P2 n1 + n2] (y = x*chirp, zero past N), times W_P^{n2 k1}
//       -> A[k1][n2]                                  (coalesced 8-wide rows)
//   KB  k_large_rows<MAIN>: per row k1, FFT_P2 over n2 -> Y[k1 + P1 k2],
//       times Ht[k1][k2] = H[k1 + P1 k2]/P, conj, FFT_P2 over k2, times
//       W_P^{k1 c} -> B[k1][c]       (forward step 3 + inverse step 1 fused:
//       the spectrum never leaves the CTA)
//   KC  k_large_cols<INV>: per tile of 8 columns c, FFT_P1 over k1 of
//       B[k1][c] -> G[c + P2 d]; X[m] = chirp[m] * conj(G[m]) for m < M.
// The plan builds Ht with KA (on h) + k_large_rows<SPECTRUM>.
//
// The same two kernels run the α-FFT itself (method fft) at sizes past one
// CTA, α = 1/r with r a power of two (the reference's plan() rule,
// fastpath.py:97-101), N = P1 x P2, one output residue c < r per launch pair:
// bins m = c + r d, d = d1 + P1 d2, n = P2 n1 + n2,
//   X[c + r d] = Σ_{n2} W_{P2}^{d2 n2} · W_{rN}^{(c + r d1) n2}
//                · Σ_{n1} W_{P1}^{d1 n1} · W_{rP1}^{c n1} · x[P2 n1 + n2]
//   KA  k_large_cols<AFFT>: per column n2, × W_{rP1}^{c n1} (the α pre-twiddle's
//       n1 part), FFT_P1 over n1, × W_{rN}^{(c + r d1) n2} -> A[d1][n2]
//   KB  k_large_rows<AFFT>: per row d1, FFT_P2 over n2 -> X[c + r(d1 + P1 d2)]
//       for the d2 with m < M (the recursion's even/odd split per residue,
//       DESIGN.md §2; twiddles exact: one two-level lookup of W_{rN}).
#pragma once

#include "asx_kernels.cuh"

namespace asx {

#ifndef ASX_COL_TILE
#define ASX_COL_TILE 4
#endif
// columns per CTA in the column kernels: 4 x 16 B = 64 B row segments (two
// full sectors); small enough for two CTAs per SM, so one CTA's gather
// latency overlaps the other's butterflies (8 columns: 128 B rows but one
// CTA per SM, config 2 0.163 ms per column pass)
constexpr int kColTile = ASX_COL_TILE;
#ifndef ASX_COL_SKEW
#define ASX_COL_SKEW 1  // column stride of the tile skewed so the kColTile columns of a row fall into distinct bank groups
#endif
#ifndef ASX_COL_TWCHAIN
#define ASX_COL_TWCHAIN 1  // column-pass twiddles W^{(t + NT i) col} = W^{t col} (W^{NT col})^i: 2 table lookups per thread and tile instead of R
#endif
// Column stride (elements of elem_bytes) >= base: the tile is filled and drained by kColTile threads per row
// (tau * CS + row), so tau * CS must step through the eight 16-byte bank groups (base strides are multiples of 8:
// a 4-way conflict on every tile access, 40 % of the column passes' shared-memory wavefronts).
constexpr int col_stride(int base, int elem_bytes) {
#if ASX_COL_SKEW
  const int unit = 16 / elem_bytes > 0 ? 16 / elem_bytes : 1;
  const int mod = 8 * unit, target = unit * (8 / kColTile > 0 ? 8 / kColTile : 1);
  return base + ((target - base % mod) + mod) % mod;
#else
  return base;
#endif
}
template <int NT>
constexpr int col_minb() {
  return (1024 / (NT * kColTile)) < 1 ? 1 : (1024 / (NT * kColTile)) > 16 ? 16 : (1024 / (NT * kColTile));
}

struct LParams {
  const void* x;  // input row (real or complex), N samples
  int real_in;
  int64_t n, m;
  void* X;              // output row, M bins
  const void* chirp;    // chirp[k], k < max(N, M)
  const void* h;        // KA on the kernel table (plan time): complex h[P]
  void* A;              // workspace P complex (row-major [P1][P2])
  const void* Ht;       // spectrum table [P1][P2]
  void* Hout;           // plan time: spectrum output
  const void* twP1;     // two-level W_P1
  const void* twP2;     // two-level W_P2
  const void* twBig;    // two-level W_P
  int lfBig;
  double scale;         // plan time: 1/P
  int64_t P;            // P1 * P2
  int64_t P2;           // row length (row stride of A / Ht)
  int64_t r, c;         // α-FFT modes: density r (power of two), residue c; twBig = W_{rN}
  int64_t nsig;         // signals per launch (batched: workspace [nsig][P], x / X rows at xs / Xs)
  int64_t xs, Xs;       // row strides of x and X (elements)
};

template <typename C>
__device__ __forceinline__ C tw_big(const C* tw, uint64_t k, int lf) {
  const C f = __ldg(tw + (k & ((uint64_t(1) << lf) - 1)));
  const C c = __ldg(tw + (uint64_t(1) << lf) + (k >> lf));
  return cmul(f, c);
}

// v[i] *= W^{e0 + i es}, i < R (W = the two-level table's root, exponents reduced by mask): base, step and
// step^4 are exact lookups, every other power at most R / 4 + 1 further products on top of them (FP64 only: the
// chain's rounding, a few 1e-16, is far inside the 1e-10 bound; complex64 keeps one lookup per element).
// Replaces 2 R scattered 16-byte table loads per thread by 6 at the same number of FP64 operations.
template <typename C, int R>
__device__ __forceinline__ void tw_chain_apply(C (&v)[R], const C* tw, uint64_t e0, uint64_t es, uint64_t mask, int lf) {
  const C b = tw_big(tw, e0 & mask, lf);
  if constexpr (R < 4) {
    v[0] = cmul(v[0], b);
    if constexpr (R == 2) v[1] = cmul(v[1], cmul(b, tw_big(tw, es & mask, lf)));
  } else {
    const C s1 = tw_big(tw, es & mask, lf), s2 = cmul(s1, s1), s3 = cmul(s2, s1);
    C wh = b;
    C s4 = b;
    if constexpr (R > 4) s4 = tw_big(tw, (4 * es) & mask, lf);
#pragma unroll
    for (int hi = 0; hi < R / 4; ++hi) {
      v[4 * hi] = cmul(v[4 * hi], wh);
      v[4 * hi + 1] = cmul(v[4 * hi + 1], cmul(wh, s1));
      v[4 * hi + 2] = cmul(v[4 * hi + 2], cmul(wh, s2));
      v[4 * hi + 3] = cmul(v[4 * hi + 3], cmul(wh, s3));
      if (hi + 1 < R / 4) wh = cmul(wh, s4);
    }
  }
}

#ifdef ASX_COLS_TIMELINE
#define COLS_TL(i) do { if (threadIdx.x == 0 && blockIdx.x == 5) tl_[i] = clock64(); } while (0)
#define COLS_TL_PRINT() do { if (threadIdx.x == 0 && blockIdx.x == 5 && un == blockIdx.x + 2 * gridDim.x) \
  printf("cols mode %d: gather %lld sync %lld vread %lld fft %lld tw %lld sts %lld out %lld total %lld\n", MODE, tl_[1]-tl_[0], tl_[2]-tl_[1], tl_[3]-tl_[2], tl_[4]-tl_[3], tl_[5]-tl_[4], tl_[6]-tl_[5], tl_[7]-tl_[6], tl_[7]-tl_[0]); } while (0)
#else
#define COLS_TL(i)
#define COLS_TL_PRINT()
#endif
enum { COL_FWD_SIGNAL = 0, COL_FWD_TABLE = 1, COL_INV_OUT = 2, COL_AFFT = 3 };

template <typename Real, int P1>
struct ColCfg {
  static constexpr int R = P1 < 8 ? P1 : 8;
  static constexpr int NT = P1 / R;
  using E = Fft<Real, P1, NT>;
  static constexpr int CS = col_stride(E::SMEM_ELEMS > P1 + (P1 >> E::LPAD) ? E::SMEM_ELEMS : P1 + (P1 >> E::LPAD),
                                       int(sizeof(typename CT<Real>::T)));
  static constexpr size_t SMEM = (size_t(kColTile) * CS + E::TAB_ELEMS + 2) * sizeof(typename CT<Real>::T) + 16;
};

// 8 teams of NT threads, one column each; the tile passes through the teams'
// shared buffers on the way in and out so HBM sees 128 B row segments.
template <typename Real, int P1, int NT, int MODE>
__global__ void __launch_bounds__(NT* kColTile, col_minb<NT>()) k_large_cols(LParams p) {
  using E = Fft<Real, P1, NT>;
  using C = typename CT<Real>::T;
  constexpr int R = E::R;
  constexpr int THREADS = NT * kColTile;
  const int64_t P2 = p.P2;
  // twBig period: P (chirp), r N (α-FFT; both powers of two)
  const uint64_t Pmask = MODE == COL_AFFT ? uint64_t(p.r * p.P - 1) : uint64_t(p.P - 1);
  constexpr int CS = ColCfg<Real, P1>::CS;  // per-column stride
  extern __shared__ __align__(128) unsigned char smraw[];
  C* smbase = reinterpret_cast<C*>(smraw);
  const int team = threadIdx.x / NT, t = threadIdx.x % NT;
  C* sm = smbase + team * CS;
  C* tabp = smbase + kColTile * CS;
  const typename E::TwRegs tr = E::make_tw(t, reinterpret_cast<const C*>(p.twP1), tabp, threadIdx.x, THREADS);
  typename E::XSync xs;
  E::xs_init(xs, reinterpret_cast<uint64_t*>(tabp + E::TAB_ELEMS + (E::TAB_ELEMS & 1)), THREADS);

  // persistent over column tiles: the per-CTA twiddle setup (make_tw, FP64
  // sincospi seeds) is paid once per CTA instead of once per tile
  const int ntiles = int(P2 / kColTile);
#ifdef ASX_COLS_TIMELINE
  long long tl_[8];
#endif
  const int64_t units = int64_t(ntiles) * p.nsig;  // (signal, column tile) pairs of the group
#pragma unroll 1
  for (int64_t un = blockIdx.x; un < units; un += gridDim.x) {
    const int64_t g = un / ntiles;
    const int col0 = int(un - g * ntiles) * kColTile;
    const void* xg = static_cast<const char*>(p.x) + g * p.xs * (p.real_in ? sizeof(Real) : sizeof(C));
    C* const Ag = reinterpret_cast<C*>(p.A) + g * p.P;
    C* const Xg = reinterpret_cast<C*>(p.X) + g * p.Xs;
    __syncthreads();  // the previous tile's write-out reads of smbase are done
    COLS_TL(0);
    // ---- gather the column tile: kColTile threads per row, rows strided.  All of a thread's loads are issued
    // before the first use (one HBM latency per tile instead of one per row: the bounds checks otherwise keep
    // the compiler from hoisting the loads of later rows over the shared-memory stores of earlier ones) ----
    {
      constexpr int RSTEP = THREADS / kColTile, G = P1 / RSTEP;  // rows per thread
      const int tau = threadIdx.x & (kColTile - 1), row0 = threadIdx.x / kColTile;
      const int64_t idx0 = int64_t(row0) * P2 + col0 + tau, istep = int64_t(RSTEP) * P2;
      C val[G];
      if constexpr (MODE == COL_FWD_SIGNAL) {
        // y[n] = x[n] * chirp[n], zero past N
        const C* ch = reinterpret_cast<const C*>(p.chirp);
        C cw[G];
#pragma unroll
        for (int k = 0; k < G; ++k) {
          const int64_t idx = idx0 + k * istep;
          cw[k] = idx < p.n ? __ldg(ch + idx) : mk(Real(0), Real(0));
        }
        if (p.real_in) {
          Real xr[G];
#pragma unroll
          for (int k = 0; k < G; ++k) {
            const int64_t idx = idx0 + k * istep;
            xr[k] = idx < p.n ? __ldg(reinterpret_cast<const Real*>(xg) + idx) : Real(0);
          }
#pragma unroll
          for (int k = 0; k < G; ++k) val[k] = cmul(mk(xr[k], Real(0)), cw[k]);
        } else {
#pragma unroll
          for (int k = 0; k < G; ++k) {
            const int64_t idx = idx0 + k * istep;
            val[k] = idx < p.n ? __ldg(reinterpret_cast<const C*>(xg) + idx) : mk(Real(0), Real(0));
          }
#pragma unroll
          for (int k = 0; k < G; ++k) val[k] = cmul(val[k], cw[k]);
        }
      } else if constexpr (MODE == COL_FWD_TABLE) {
#pragma unroll
        for (int k = 0; k < G; ++k) val[k] = __ldg(reinterpret_cast<const C*>(p.h) + idx0 + k * istep);
      } else if constexpr (MODE == COL_AFFT) {
        // x[P2 n1 + n2] × W_{rP1}^{c n1} = W_{rN}^{c n1 P2}
        if (p.real_in) {
#pragma unroll
          for (int k = 0; k < G; ++k)
            val[k] = mk(__ldg(reinterpret_cast<const Real*>(xg) + idx0 + k * istep), Real(0));
        } else {
#pragma unroll
          for (int k = 0; k < G; ++k) val[k] = __ldg(reinterpret_cast<const C*>(xg) + idx0 + k * istep);
        }
        if (p.c) {
#pragma unroll
          for (int k = 0; k < G; ++k)
            val[k] = cmul(val[k], tw_big(reinterpret_cast<const C*>(p.twBig),
                                         (uint64_t(p.c) * uint64_t(row0 + k * RSTEP) * uint64_t(P2)) & Pmask, p.lfBig));
        }
      } else {
#pragma unroll
        for (int k = 0; k < G; ++k) val[k] = __ldg(Ag + idx0 + k * istep);  // B[k1][c], row = k1
      }
#pragma unroll
      for (int k = 0; k < G; ++k) smbase[tau * CS + E::pad(row0 + k * RSTEP)] = val[k];
    }
    COLS_TL(1);
    __syncthreads();
    COLS_TL(2);
    C v[R];
  #pragma unroll
    for (int i = 0; i < R; ++i) v[i] = sm[E::pad(t + NT * i)];
    __syncthreads();       // tile reads done before the transform reuses sm
    COLS_TL(3);
    E::run(v, sm, t, tr, xs);
    COLS_TL(4);
    const int col = col0 + team;
    if constexpr (ASX_COL_TWCHAIN && sizeof(Real) == 8 && MODE != COL_INV_OUT) {
      // twiddle W^{e0 + i es}: W_P^{n2 k1}, k1 = t + NT i (chirp), W_{rN}^{(c + r d1) n2}, d1 = t + NT i (α-FFT);
      const C* tw = reinterpret_cast<const C*>(p.twBig);
      const uint64_t e0 = MODE == COL_AFFT ? (uint64_t(p.c) + uint64_t(p.r) * uint64_t(t)) * uint64_t(col)
                                           : uint64_t(t) * uint64_t(col);
      const uint64_t es = (MODE == COL_AFFT ? uint64_t(p.r) : uint64_t(1)) * uint64_t(NT) * uint64_t(col);
      tw_chain_apply<C, R>(v, tw, e0, es, Pmask, p.lfBig);
    } else if constexpr (MODE == COL_AFFT) {
      // twiddle W_{rN}^{(c + r d1) n2}, d1 = t + NT*i
  #pragma unroll
      for (int i = 0; i < R; ++i) {
        const uint64_t e = (uint64_t(p.c) + uint64_t(p.r) * uint64_t(t + NT * i)) * uint64_t(col);
        v[i] = cmul(v[i], tw_big(reinterpret_cast<const C*>(p.twBig), e & Pmask, p.lfBig));
        if ((i % ASX_FENCE_CHUNK) == ASX_FENCE_CHUNK - 1) reg_fence();
      }
    } else if constexpr (MODE != COL_INV_OUT) {
      // twiddle W_P^{n2 k1}, k1 = t + NT*i
  #pragma unroll
      for (int i = 0; i < R; ++i) {
        const uint64_t k1 = uint64_t(t + NT * i);
        v[i] = cmul(v[i], tw_big(reinterpret_cast<const C*>(p.twBig), (k1 * uint64_t(col)) & Pmask, p.lfBig));
        if ((i % ASX_FENCE_CHUNK) == ASX_FENCE_CHUNK - 1) reg_fence();
      }
    }
    COLS_TL(5);
    __syncthreads();
  #pragma unroll
    for (int i = 0; i < R; ++i) sm[E::pad(t + NT * i)] = v[i];
    __syncthreads();
    COLS_TL(6);
    {
      constexpr int RSTEP = THREADS / kColTile, G = P1 / RSTEP;
      const int tau = threadIdx.x & (kColTile - 1), row0 = threadIdx.x / kColTile;
      if constexpr (MODE != COL_INV_OUT) {
#pragma unroll
        for (int k = 0; k < G; ++k) {
          const int row = row0 + k * RSTEP;
          Ag[int64_t(row) * P2 + col0 + tau] = smbase[tau * CS + E::pad(row)];
        }
      } else {
        // X[m] = conj(G[m]) chirp[m], m = c + P2 d < M: the chirp loads of all rows first
        const C* ch = reinterpret_cast<const C*>(p.chirp);
        const int64_t mm0 = int64_t(col0 + tau) + P2 * row0, mstep = P2 * RSTEP;
        C cw[G];
#pragma unroll
        for (int k = 0; k < G; ++k) cw[k] = mm0 + k * mstep < p.m ? __ldg(ch + mm0 + k * mstep) : mk(Real(0), Real(0));
#pragma unroll
        for (int k = 0; k < G; ++k) {
          const int64_t mm = mm0 + k * mstep;
          if (mm < p.m) Xg[mm] = cmul(cconj(smbase[tau * CS + E::pad(row0 + k * RSTEP)]), cw[k]);
        }
      }
    }
    COLS_TL(7); COLS_TL_PRINT();
  }
}

enum { ROW_SPECTRUM = 0, ROW_MAIN = 1, ROW_MAIN_LOCAL = 2, ROW_AFFT = 3 };  // 2: k_large_rows_local (asx_chirp_local128.cuh)

__device__ __forceinline__ void prefetch_l2_bulk(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// Persistent over rows (grid <= #SMs): while row k1 is transformed, the next
// row of A (and of Ht) is prefetched into L2, so the row loads of one CTA per
// SM wait on L2 instead of HBM.
template <typename Real, int P2, int NT, int MODE>
__global__ void __launch_bounds__(NT, 1) k_large_rows(LParams p) {
  using E = Fft<Real, P2, NT>;
  using C = typename CT<Real>::T;
  constexpr int R = E::R;
  constexpr uint32_t ROW_BYTES = uint32_t(P2) * sizeof(C);
  const uint64_t Pmask = uint64_t(p.P - 1);
  extern __shared__ __align__(128) unsigned char smraw[];
  C* sm = reinterpret_cast<C*>(smraw);
  const int t = threadIdx.x;
  const int rows = int(p.P / P2);
  const int64_t urows = int64_t(rows) * p.nsig;  // the group's workspaces are one [nsig * rows][P2] matrix
  const typename E::TwRegs tr =
      E::make_tw(t, reinterpret_cast<const C*>(p.twP2), sm + E::SMEM_ELEMS, threadIdx.x, NT);
  typename E::XSync xs;
  E::xs_init(xs, reinterpret_cast<uint64_t*>(sm + E::SMEM_ELEMS + E::TAB_ELEMS + (E::TAB_ELEMS & 1)), NT);
  __syncthreads();
#pragma unroll 1
  for (int64_t ur = blockIdx.x; ur < urows; ur += gridDim.x) {
    const int k1 = int(ur % rows);
    const int64_t g = ur / rows;
    if (t == 0 && ur + int64_t(gridDim.x) < urows) {
      const int64_t nr = ur + int64_t(gridDim.x);
      prefetch_l2_bulk(reinterpret_cast<const C*>(p.A) + nr * P2, ROW_BYTES);
      if (MODE == ROW_MAIN) prefetch_l2_bulk(reinterpret_cast<const C*>(p.Ht) + (nr % rows) * P2, ROW_BYTES);
    }
    C* row = reinterpret_cast<C*>(p.A) + ur * P2;
    C v[R];
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = row[t + NT * i];
    if constexpr (MODE == ROW_SPECTRUM) {
      E::run(v, sm, t, tr, xs);
      C* out = reinterpret_cast<C*>(p.Hout) + int64_t(k1) * P2;
      const Real s = Real(p.scale);
#pragma unroll
      for (int i = 0; i < R; ++i) out[t + NT * i] = mk(v[i].x * s, v[i].y * s);
    } else if constexpr (MODE == ROW_AFFT) {
      // X[c + r (d1 + P1 d2)], d1 = k1, d2 = t + NT*i; bins past M are not stored
      E::run(v, sm, t, tr, xs);
      const int64_t P1 = p.P / P2;
      C* X = reinterpret_cast<C*>(p.X) + g * p.Xs;
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int64_t mm = p.c + p.r * (int64_t(k1) + P1 * int64_t(t + NT * i));
        if (mm < p.m) X[mm] = v[i];
      }
    } else {
      const C* ht = reinterpret_cast<const C*>(p.Ht) + int64_t(k1) * P2;
      // one FFT body, two trips (forward step 3, then inverse step 1)
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        E::run(v, sm, t, tr, xs);
        if (half == 0) {
#pragma unroll
          for (int i = 0; i < R; ++i) {
            v[i] = cconj(cmul(v[i], __ldg(ht + t + NT * i)));
            if ((i % ASX_FENCE_CHUNK) == ASX_FENCE_CHUNK - 1) reg_fence();
          }
        }
      }
      if constexpr (ASX_COL_TWCHAIN && sizeof(Real) == 8) {
        // W_P^{k1 c}, c = t + NT i
        tw_chain_apply<C, R>(v, reinterpret_cast<const C*>(p.twBig), uint64_t(k1) * uint64_t(t),
                             uint64_t(k1) * uint64_t(NT), Pmask, p.lfBig);
#pragma unroll
        for (int i = 0; i < R; ++i) row[t + NT * i] = v[i];
      } else {
#pragma unroll
        for (int i = 0; i < R; ++i) {
          const uint64_t c = uint64_t(t + NT * i);
          row[t + NT * i] =
              cmul(v[i], tw_big(reinterpret_cast<const C*>(p.twBig), (uint64_t(k1) * c) & Pmask, p.lfBig));
          if ((i % ASX_FENCE_CHUNK) == ASX_FENCE_CHUNK - 1) reg_fence();
        }
      }
    }
  }
}

// h[j] = conj(chirp[j]) (j < M), conj(chirp[P-j]) (P-j < N), else 0.
template <typename Real>
static __global__ void k_fill_h(void* h, const void* chirp, int64_t P, int64_t n, int64_t m) {
  using C = typename CT<Real>::T;
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < P; j += int64_t(gridDim.x) * blockDim.x) {
    C v = mk(Real(0), Real(0));
    if (j < m)
      v = cconj(__ldg(reinterpret_cast<const C*>(chirp) + j));
    else if (P - j < n)
      v = cconj(__ldg(reinterpret_cast<const C*>(chirp) + (P - j)));
    reinterpret_cast<C*>(h)[j] = v;
  }
}

}  // namespace asx

// asx_kernels.cuh — sm_100a kernels of the α-DFT / α-FFT hot path.
//
//   k_afft    α-FFT (fastpath.py:130-181), one team per (signal, output residue)
//   k_chirp   chirp-z factorisation of the same α-DFT, one team per signal
//   k_direct  direct α-DFT as a tiled complex contraction with W[M,N]
//             (oracle.py:37-67 _reduced_product, batched)
//   plan-time table builders (exact integer argument reduction + sincospi,
//   the device restatement of oracle.py:21-23 roots_of_unity and the
//   fastpath.py:104-109 twiddle tables)
//   k_combine / k_block_sum  the reference's building blocks
//   (fastpath.py:130-151, :154-159)
#pragma once

#include "asx_engine.cuh"

#ifndef ASX_AFFT_RESEED
#define ASX_AFFT_RESEED 4  // α-FFT pre-twiddle: exact table value every N elements, chained between
#endif
#ifndef ASX_ZERO_PRUNE
#define ASX_ZERO_PRUNE 1  // chirp: compile-time zero upper half of the FFT input
#endif
#ifndef ASX_FENCE_CHUNK
#define ASX_FENCE_CHUNK 4  // table loads issued per group between compiler fences
#endif

namespace asx {

struct KParams {
  const void* x;
  int64_t xs;  // input row stride (elements)
  void* X;
  int64_t Xs;  // output row stride (complex elements)
  int64_t batch;
  int64_t n, m;
  int64_t r;     // afft: output residue classes (alpha = 1/r); 1 when folding
  int64_t fold;  // afft: folded blocks (alpha = fold, BLOCK_SUM leaf); else 1
  int real_in;
  int lfA;             // log2 of the fine part of twA
  const void* twP;     // two-level W_P table (P = inner FFT size)
  const void* twA;     // two-level W_{rN} table (α pre-twiddle)
  const void* chirp;   // chirp[k], k < max(N, M)
  const void* H;       // chirp kernel spectrum / P, P entries
  const void* W;       // direct: M x N
  int staged;          // 1: rows fetched by TMA into shared memory
  int tw_elems;        // shared twiddle elements (W_P two-level [+ W_rN two-level])
  int64_t chirp_len;   // entries of the chirp table (max(N, M))
  const void* afl;     // k_afft_local: per-thread twiddle image for tensor memory (plan time), else null
};

template <typename C>
__device__ __forceinline__ C load_in(const void* x, int64_t idx, int real_in) {
  using Real = decltype(C{}.x);
  if (real_in) return mk(__ldg(reinterpret_cast<const Real*>(x) + idx), Real(0));
  return __ldg(reinterpret_cast<const C*>(x) + idx);
}

// Input sample n of the staged row (shared memory) or straight from global.
template <typename C>
__device__ __forceinline__ C load_row(const unsigned char* stage, const void* x, int64_t row_off, int64_t n,
                                      int real_in, bool staged) {
  using Real = decltype(C{}.x);
  if (staged) {
    if (real_in) return mk(reinterpret_cast<const Real*>(stage)[n], Real(0));
    return reinterpret_cast<const C*>(stage)[n];
  }
  return load_in<C>(x, row_off + n, real_in);
}

// complex value converted to another precision (identity when equal)
template <typename To, typename From>
__device__ __forceinline__ To widen(From v) {
  if constexpr (sizeof(To) == sizeof(From))
    return v;
  else
    return mk(decltype(To{}.x)(v.x), decltype(To{}.x)(v.y));
}

// Compiler-only fence: keeps the scheduler from hoisting every table load of an
// unrolled loop at once (which would double live registers and spill).
__device__ __forceinline__ void reg_fence() { asm volatile("" ::: "memory"); }

__host__ __device__ constexpr size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Shared-memory layout of the persistent FFT-family kernels (host and device
// agree on it through this helper).
template <typename Real, int P, int NT, int KIND>
constexpr bool persist_dbuf() {
  // warp teams (NT <= 32) protect the exchange with one __syncwarp instead
  return KIND == 1 && size_t(P) * sizeof(typename CT<Real>::T) <= ASX_DBUF_MAX_BYTES && !(NT > 1 && NT <= 32);
}

template <typename Real, int P, int NT, int TPB, bool TS = false, int KR = 1, bool DBUF = false, int NSTAGE = TPB>
struct PersistLayout {
  using E = Fft<Real, P, NT, ASX_TWTAB_MAX, TS, DBUF>;
  using C = typename CT<Real>::T;
  static constexpr size_t FFT_BYTES = align_up(size_t(TPB) * KR * E::SMEM_ELEMS * sizeof(C), 128);
  __host__ __device__ static size_t stage_bytes(size_t row_bytes, bool staged) {
    return staged ? align_up(row_bytes, 128) : 0;
  }
  static constexpr size_t TAB_BYTES = align_up(size_t(E::TAB_ELEMS) * sizeof(C), 16);
  __host__ __device__ static size_t tab_off(size_t row_bytes, bool staged) {
    return FFT_BYTES + size_t(NSTAGE) * stage_bytes(row_bytes, staged);
  }
  __host__ __device__ static size_t tw_off(size_t row_bytes, bool staged) {
    return tab_off(row_bytes, staged) + TAB_BYTES;
  }
  // [fft buffers | stage rows | twiddle tables | α table | mbarriers | TMEM slot]
  __host__ __device__ static size_t total(size_t row_bytes, bool staged, size_t tw_elems) {
    return align_up(tw_off(row_bytes, staged) + tw_elems * sizeof(C), 16) + TPB * sizeof(uint64_t) + 16;
    // tail: TPB TMA mbarriers, the exchange WAR mbarrier, the TMEM address slot
  }
};

// ---------------------------------------------------------------------------
// Persistent FFT-family kernel: each NT-thread team walks its signals
// u = blockIdx.x*TPB + team, += gridDim.x*TPB.  The next signal's row is
// fetched global -> shared by a TMA bulk copy (cp.async.bulk + mbarrier)
// while the current one is transformed; twiddle tables live in shared
// memory; results leave registers straight to HBM in the io layout.
//
// KIND_AFFT — α-FFT, α = 1/r (reference DenseFactor(r), SINGLE_SAMPLE leaf)
// or α = fold (DenseFactor(1, fold), BLOCK_SUM leaf).  The reference sweeps
// the even/odd recursion level-synchronously over the whole r*N-bin
// spectrum (fastpath.py:162-181), a working set of r*N values per signal.
// Splitting the bin index m = c + r*d (c < r) turns the (rN x N) matrix into
// r independent (N x N) DFTs of the α-twiddled signal x_n * W_{rN}^{c n},
// each evaluated by the same radix-2^k even/odd recursion (fastpath.py:
// 130-151 butterflies, Rp levels fused per pass), so a team needs only N
// values of state and bins m >= M are never stored.
//
// KIND_CHIRP — chirp-z: a*m*n = a*(m^2 + n^2 - (m-n)^2)/2 turns the α-DFT into
//   X_m = chirp[m] * sum_n (x_n chirp[n]) * conj(chirp[m-n]),
//   chirp[k] = exp(-pi*i*((a k^2) mod 2dN)/(dN)),
// a linear convolution done as a P-point cyclic one (P >= N+M-1): forward
// FFT, multiply by H = FFT(h)/P, inverse FFT as conj(FFT(conj(.))).  The
// last forward pass and the first inverse pass share the io layout, so the
// spectrum never leaves registers.
// ---------------------------------------------------------------------------
enum { KIND_AFFT = 0, KIND_CHIRP = 1 };

// TMEM layout of the chirp tables (TM variant; CTA size NTH % 128 == 0): warp
// w owns lanes 32*(w%4).., column slot w/4 of CPT columns: H[t + NT*j] for
// j < R, then chirp[t + NT*j] for j < R.
template <typename Real, int NTH, int R, int SEEDCOLS = 0>
struct TmemCfg {
  static constexpr int WPC = sizeof(typename CT<Real>::T) / 4;  // 32-bit words per complex
  static constexpr int RH = R > 1 ? R / 2 : 1;                  // chirp values kept (M <= P/2)
  static constexpr int SEED_OFF = (R + RH) * WPC;
  static constexpr int CPT = SEED_OFF + SEEDCOLS;               // columns per thread
  static constexpr int CPC = 8 / WPC;                           // complex per 8-column access
  static constexpr int NEED = (NTH / 128) * CPT;
  static constexpr int NCOLS = NEED <= 32 ? 32 : NEED <= 64 ? 64 : NEED <= 128 ? 128 : NEED <= 256 ? 256 : 512;
  static constexpr bool OK = (NTH % 128 == 0) && NEED <= 512;
};

// SPLIT (α-FFT only): the TPB teams of a CTA share ONE signal and split its
// r output residues (team j takes c = j, j + TPB, ...); one TMA-staged row
// serves them all, so a CTA of TPB teams keeps staging at full occupancy.
// RS (α-FFT, small batches): the work unit is one (signal, residue) pair
// instead of a signal, so one signal's r residues run on r teams at once.
// IO (α-FFT only): the element type of x and X when it differs from the
// arithmetic type Real (complex64 plans run the recursion in FP64: samples are
// widened on load, bins rounded once on store).
template <typename Real, int P, int NT, int TPB, int KIND, int MINB, bool TM = false, int KR = 1, bool SPLIT = false,
          bool RS = false, typename IO = Real>
__global__ void __launch_bounds__(NT* TPB, MINB) k_fft_persist(KParams p) {
  static_assert(!SPLIT || (KIND == 0 && NT > 32), "SPLIT: alpha-FFT with CTA-wide team barriers");
  static_assert(KIND == 0 || sizeof(IO) == sizeof(Real), "mixed precision: alpha-FFT only");
  using CI = typename CT<IO>::T;
  constexpr bool TS = TM && KIND == KIND_CHIRP;  // last-pass twiddle seeds in TMEM too
  constexpr bool DBUF = persist_dbuf<Real, P, NT, KIND>();
  using E = Fft<Real, P, NT, ASX_TWTAB_MAX, TS, DBUF>;
  using L = PersistLayout<Real, P, NT, TPB, TS, KR, DBUF, SPLIT ? 1 : TPB>;
  constexpr int SIG_PER_CTA = SPLIT ? 1 : TPB;  // signals in flight per CTA
  using C = typename CT<Real>::T;
  constexpr int R = E::R;
  extern __shared__ __align__(128) unsigned char smraw[];
  const int team = threadIdx.x / NT, t = threadIdx.x % NT;
  const bool staged = p.staged != 0;
  const size_t row_bytes = size_t(p.n) * (p.real_in ? sizeof(IO) : sizeof(CI));
  C* fbuf = reinterpret_cast<C*>(smraw) + team * KR * E::SMEM_ELEMS;
  const int steam = SPLIT ? 0 : team;  // owner of the staged row / its mbarrier
  unsigned char* stage = smraw + L::FFT_BYTES + steam * L::stage_bytes(row_bytes, staged);
  C* twa = reinterpret_cast<C*>(smraw + L::tw_off(row_bytes, staged));  // α pre-twiddle W_{rN} (afft, r > 1)
  uint64_t* const bar0 = reinterpret_cast<uint64_t*>(
      smraw + align_up(L::tw_off(row_bytes, staged) + p.tw_elems * sizeof(C), 16));
  uint64_t* bar = bar0 + steam;

  // per-thread pass twiddles -> registers; α pre-twiddle table -> shared
  typename E::TwRegs tr =
      E::make_tw(t, reinterpret_cast<const C*>(p.twP), reinterpret_cast<C*>(smraw + L::tab_off(row_bytes, staged)),
                 threadIdx.x, NT * TPB);
  {
    const C* srca = reinterpret_cast<const C*>(p.twA);
    for (int i = threadIdx.x; i < p.tw_elems; i += NT * TPB) twa[i] = __ldg(srca + i);
  }
  // batch < 2^31 (checked on the host): 32-bit signal indices keep the
  // persistent loop's live state small next to the 2R data registers
  const int stride = int(gridDim.x) * SIG_PER_CTA;
  int u = int(blockIdx.x) * SIG_PER_CTA + (SPLIT ? 0 : team);
  const bool stage_owner = t == 0 && (!SPLIT || team == 0);
  // work units: signals, or (signal, residue) pairs when rsplit (small batches:
  // the r residues of one signal run on r teams instead of one after another)
  constexpr bool rs = KIND == KIND_AFFT && !SPLIT && RS;
  const int nres = rs ? int(p.r) : 1;
  const int batch = rs ? int(p.batch) * nres : int(p.batch);
  auto sig = [&](int unit) { return rs ? unit / nres : unit; };
  const int iters = (batch + stride - 1) / stride;
  if (staged && stage_owner) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  typename E::XSync xs;
  E::xs_init(xs, bar0 + TPB, NT * TPB);
  __syncthreads();
  if (staged && stage_owner && u < batch) {
    mbar_expect_tx(bar, (uint32_t)row_bytes);
    tma_load_1d(stage, static_cast<const unsigned char*>(p.x) + int64_t(sig(u)) * p.xs * (row_bytes / p.n),
                (uint32_t)row_bytes, bar);
  }
  uint32_t phase = 0;
  const C* chirp = reinterpret_cast<const C*>(p.chirp);
  const C* H = reinterpret_cast<const C*>(p.H);
  using TMC = TmemCfg<Real, NT * TPB, R, E::TSEED_COLS>;
  uint32_t tbase = 0;
  uint32_t& tmem_slot = *reinterpret_cast<uint32_t*>(bar0 + TPB + 1);  // after the mbarriers
  if constexpr (TM) {
    static_assert(TMC::OK, "TMEM tables need a CTA of 128k threads within 512 columns");
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc(&tmem_slot, TMC::NCOLS);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    tbase = tmem_slot + (uint32_t(32 * (warp & 3)) << 16) + uint32_t((warp >> 2) * TMC::CPT);
#pragma unroll
    for (int j0 = 0; j0 < R; j0 += TMC::CPC) {
      uint32_t wh[8], wc[8];
#pragma unroll
      for (int k = 0; k < TMC::CPC; ++k) {
        const int idx = t + NT * (j0 + k);
        c_to_words(__ldg(H + idx), &wh[k * TMC::WPC]);
        c_to_words((j0 + k < TMC::RH && idx < p.chirp_len) ? __ldg(chirp + idx) : mk(Real(0), Real(0)),
                   &wc[k * TMC::WPC]);
      }
      tmem_st8(tbase + j0 * TMC::WPC, wh);
      if (j0 < TMC::RH) tmem_st8(tbase + (R + j0) * TMC::WPC, wc);
    }
    E::store_tmem_seeds(t, tbase + TMC::SEED_OFF);
    tr.tseed = tbase + TMC::SEED_OFF;
    tmem_wait_st();
  }
  // chirp / kernel-spectrum value j of this thread (TMEM or L2)
  auto tab_chunk = [&](int which, int j0, C (&out)[TMC::CPC]) {
    if constexpr (TM) {
      uint32_t w[8];
      tmem_ld8(tbase + (which * R + j0) * TMC::WPC, w);
#pragma unroll
      for (int k = 0; k < TMC::CPC; ++k) out[k] = words_to_c(&w[k * TMC::WPC], (C*)nullptr);
    } else {
#pragma unroll
      for (int k = 0; k < TMC::CPC; ++k) {
        const int idx = t + NT * (j0 + k);
        out[k] = mk(Real(0), Real(0));
        if (j0 + k < R)
          out[k] = which == 0 ? __ldg(H + idx) : (idx < p.chirp_len ? __ldg(chirp + idx) : mk(Real(0), Real(0)));
      }
    }
  };

#pragma unroll 1
  for (int it = 0; it < iters; ++it, u += stride) {
    const bool live = u < batch;
    const int64_t row_off = int64_t(sig(u)) * p.xs;
    if constexpr (KIND == KIND_CHIRP) {
      C v[R];
      if (staged && live) {
        mbar_wait(bar, phase);
        phase ^= 1;
      }
      // the plan guarantees P >= 2N: elements t + NT*i with i >= R/2 are the
      // zero padding, known at compile time (first pass folds them away)
#pragma unroll
      for (int i = 0; i < R; ++i) v[i] = mk(Real(0), Real(0));
      constexpr int RIN = (ASX_ZERO_PRUNE && R > 1) ? R / 2 : R;
#pragma unroll
      for (int j0 = 0; j0 < RIN; j0 += (TMC::CPC < RIN ? TMC::CPC : RIN)) {
        C cw[TMC::CPC];
        tab_chunk(1, j0, cw);
        if (staged && !p.real_in && p.n >= NT * RIN && live) {  // full staged row: no per-element checks
#pragma unroll
          for (int k = 0; k < TMC::CPC && j0 + k < RIN; ++k)
            v[j0 + k] = cmul(reinterpret_cast<const C*>(stage)[t + NT * (j0 + k)], cw[k]);
        } else {
#pragma unroll
          for (int k = 0; k < TMC::CPC && j0 + k < RIN; ++k) {
            const int nn = t + NT * (j0 + k);
            if (live && nn < p.n) v[j0 + k] = cmul(load_row<C>(stage, p.x, row_off, nn, p.real_in, staged), cw[k]);
          }
        }
      }
      if (staged) {
        E::team_sync();  // the whole row has been consumed (by this team)
        if (t == 0 && u + stride < batch) {
          fence_proxy_async();
          mbar_expect_tx(bar, (uint32_t)row_bytes);
          tma_load_1d(stage, static_cast<const unsigned char*>(p.x) + int64_t(u + stride) * p.xs * (row_bytes / p.n),
                      (uint32_t)row_bytes, bar);
        }
      }
      // forward FFT, pointwise kernel spectrum, inverse FFT: one FFT body in
      // a 2-trip loop so only one copy of the transform is register-allocated
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        E::run(v, fbuf, t, tr, xs);
        if (half == 0) {
#pragma unroll
          for (int j0 = 0; j0 < R; j0 += TMC::CPC) {
            C hw[TMC::CPC];
            tab_chunk(0, j0, hw);
#pragma unroll
            for (int k = 0; k < TMC::CPC && j0 + k < R; ++k) v[j0 + k] = cconj(cmul(v[j0 + k], hw[k]));
          }
        }
      }
      {
        // table loads stay outside `live`: tcgen05.ld is warp-collective and a
        // warp may span several teams when NT < 32
        C* X = reinterpret_cast<C*>(p.X) + int64_t(u) * p.Xs;
        constexpr int ROUT = TM ? TMC::RH : R;  // TM launches need M <= P/2
#pragma unroll
        for (int j0 = 0; j0 < ROUT; j0 += (TMC::CPC < ROUT ? TMC::CPC : ROUT)) {
          C cw[TMC::CPC];
          tab_chunk(1, j0, cw);
          if (p.m >= NT * ROUT && live) {
#pragma unroll
            for (int k = 0; k < TMC::CPC && j0 + k < ROUT; ++k) X[t + NT * (j0 + k)] = cmul(cconj(v[j0 + k]), cw[k]);
          } else {
#pragma unroll
            for (int k = 0; k < TMC::CPC && j0 + k < ROUT; ++k) {
              const int mm = t + NT * (j0 + k);
              if (live && mm < p.m) X[mm] = cmul(cconj(v[j0 + k]), cw[k]);
            }
          }
        }
      }
    } else {
      if (staged && live) {
        mbar_wait(bar, phase);
        phase ^= 1;
      }
      // KR output residues at a time: their transforms share twiddles and
      // barriers and interleave in the pipeline (ILP)
      // uniform trip count over the CTA (the team barriers are CTA-wide)
      const int cbeg = rs ? u % nres : 0;
      const int64_t cend = rs ? int64_t(cbeg + 1) : p.r;
      for (int cb = cbeg; cb < cend; cb += KR * (SPLIT ? TPB : 1)) {
        const int c0 = cb + (SPLIT ? team * KR : 0);
        C v[KR][R];
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          const int c = c0 + k;
          // W_{rN}^{c n}, n = t + NT*i: base W^{c t} times step W^{c NT} chained
          // over i, re-seeded from the shared table every ASX_AFFT_RESEED steps.
          C wst = mk(Real(1), Real(0)), wc = wst;
          if (c != 0 && c < p.r) {
            wst = tw_lookup_rt(twa, c * NT, p.lfA);
            wc = tw_lookup_rt(twa, c * t, p.lfA);
          }
#pragma unroll
          for (int i = 0; i < R; ++i) {
            const int nn = t + NT * i;
            C val = mk(Real(0), Real(0));
            if (live && c < p.r) {
              val = widen<C>(load_row<CI>(stage, p.x, row_off, nn, p.real_in, staged));
              for (int s = 1; s < p.fold; ++s)
                val = cadd(val, widen<C>(load_row<CI>(stage, p.x, row_off, nn + int64_t(s) * P, p.real_in, staged)));
            }
            if (c != 0) {
              if (i > 0) wc = ((i % ASX_AFFT_RESEED) == 0) ? tw_lookup_rt(twa, c * nn, p.lfA) : cmul(wc, wst);
              val = cmul(val, wc);
            }
            v[k][i] = val;
          }
        }
        if (staged && cb + KR * (SPLIT ? TPB : 1) >= cend) {
          if constexpr (SPLIT)
            __syncthreads();  // every team has consumed the shared row
          else
            E::team_sync();
          if (stage_owner && u + stride < batch) {
            fence_proxy_async();
            mbar_expect_tx(bar, (uint32_t)row_bytes);
            tma_load_1d(stage,
                        static_cast<const unsigned char*>(p.x) + int64_t(sig(u + stride)) * p.xs * (row_bytes / p.n),
                        (uint32_t)row_bytes, bar);
          }
        }
        E::template run<KR>(v, fbuf, t, tr, xs);
        if (live) {
          CI* X = reinterpret_cast<CI*>(p.X) + int64_t(sig(u)) * p.Xs;
          const int64_t period = p.r * P;
#pragma unroll
          for (int k = 0; k < KR; ++k) {
            const int c = c0 + k;
            if (c >= p.r) continue;
#pragma unroll
            for (int i = 0; i < R; ++i) {
              const int d = t + NT * i;
              for (int64_t mm = c + p.r * d; mm < p.m; mm += period) X[mm] = widen<CI>(v[k][i]);
            }
          }
        }
      }
    }
  }
  if constexpr (TM) {
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    if ((threadIdx.x >> 5) == 0) tmem_dealloc(tmem_slot, TMC::NCOLS);
  }
}

// ---------------------------------------------------------------------------
// Direct α-DFT: X[b, m] = sum_n x[b, n] * W[m, n], a 64x64 (signals x bins)
// CTA tile, K-step 16, 4x4 complex micro-tile per thread (FFMA / DFMA).
// W is the plan's exactly-reduced matrix (oracle.py:26-34 semantics).
// ---------------------------------------------------------------------------
template <typename Real>
__global__ void __launch_bounds__(256) k_direct(KParams p) {
  using C = typename CT<Real>::T;
  constexpr int BM = 64, BN = 64, BK = 16;
  __shared__ C xs_t[BK][BM + 1];
  __shared__ C ws_t[BK][BN + 1];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t b0 = int64_t(blockIdx.y) * BM;
  const int64_t m0 = int64_t(blockIdx.x) * BN;
  const C* W = reinterpret_cast<const C*>(p.W);
  C acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = mk(Real(0), Real(0));

  for (int64_t k0 = 0; k0 < p.n; k0 += BK) {
#pragma unroll
    for (int e = 0; e < (BM * BK) / 256; ++e) {
      const int idx = tid + 256 * e;
      const int s = idx / BK, k = idx % BK;
      const int64_t bb = b0 + s, kk = k0 + k;
      C val = mk(Real(0), Real(0));
      if (bb < p.batch && kk < p.n) val = load_in<C>(p.x, bb * p.xs + kk, p.real_in);
      xs_t[k][s] = val;
      const int64_t mm = m0 + s;
      C w = mk(Real(0), Real(0));
      if (mm < p.m && kk < p.n) w = __ldg(W + mm * p.n + kk);
      ws_t[k][s] = w;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      C a[4], w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = xs_t[k][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) w[j] = ws_t[k][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[i][j].x = fma(a[i].x, w[j].x, fma(-a[i].y, w[j].y, acc[i][j].x));
          acc[i][j].y = fma(a[i].x, w[j].y, fma(a[i].y, w[j].x, acc[i][j].y));
        }
    }
    __syncthreads();
  }
  C* X = reinterpret_cast<C*>(p.X);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t bb = b0 + ty + 16 * i;
    if (bb >= p.batch) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t mm = m0 + tx + 16 * j;
      if (mm < p.m) X[bb * p.Xs + mm] = acc[i][j];
    }
  }
}

// Direct α-DFT for a handful of signals (batch <= kDirectSmallBatch): a
// matrix-vector product per signal.  Four warps share one output bin m, each
// streaming a quarter of row m of W (coalesced, lanes over n) and reusing it
// for every signal of the batch; partial sums meet in shared memory.  The
// 64-signal tile of k_direct would leave 63/64 of its work idle at batch 1
// (config 0: 0.275 ms).
constexpr int kDirectSmallBatch = 8;

template <typename Real>
__global__ void __launch_bounds__(256) k_direct_small(KParams p) {
  using C = typename CT<Real>::T;
  constexpr int NB = kDirectSmallBatch, WPB = 4;  // warps per bin
  __shared__ C part[8][NB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, q = warp % WPB;
  const int64_t mm = int64_t(blockIdx.x) * (8 / WPB) + warp / WPB;
  const int nb = int(p.batch);
  C acc[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) acc[b] = mk(Real(0), Real(0));
  if (mm < p.m) {
    const C* W = reinterpret_cast<const C*>(p.W) + mm * p.n;
    const int64_t k0 = (p.n * q) / WPB, k1 = (p.n * (q + 1)) / WPB;
#pragma unroll 4
    for (int64_t k = k0 + lane; k < k1; k += 32) {
      const C w = __ldg(W + k);
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        if (b < nb) {
          const C xv = load_in<C>(p.x, int64_t(b) * p.xs + k, p.real_in);
          acc[b].x = fma(xv.x, w.x, fma(-xv.y, w.y, acc[b].x));
          acc[b].y = fma(xv.x, w.y, fma(xv.y, w.x, acc[b].y));
        }
      }
    }
  }
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    Real ax = acc[b].x, ay = acc[b].y;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ax += __shfl_xor_sync(0xffffffffu, ax, o);
      ay += __shfl_xor_sync(0xffffffffu, ay, o);
    }
    if (lane == 0) part[warp][b] = mk(ax, ay);
  }
  __syncthreads();
  if (q == 0 && lane < nb && mm < p.m) {
    C s = part[warp][lane];
#pragma unroll
    for (int i = 1; i < WPB; ++i) s = cadd(s, part[warp + i][lane]);
    reinterpret_cast<C*>(p.X)[int64_t(lane) * p.Xs + mm] = s;
  }
}

// ----------------------------- plan-time tables ----------------------------

__device__ __forceinline__ uint64_t mulmod(uint64_t a, uint64_t b, uint64_t L) {
  return (uint64_t)(((unsigned __int128)a * b) % L);
}

__device__ __forceinline__ void store_c(void* out, int64_t i, double re, double im, int dbl) {
  if (dbl)
    reinterpret_cast<double2*>(out)[i] = make_double2(re, im);
  else
    reinterpret_cast<float2*>(out)[i] = make_float2((float)re, (float)im);
}

// out[k] = W_L^{(k*step) mod L} = exp(-2*pi*i*((k*step) mod L)/L), k < count.
static __global__ void k_fill_roots(void* out, int64_t count, uint64_t step, uint64_t L, int dbl) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < count;
       k += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t j = mulmod((uint64_t)k, step, L);
    double s, c;
    sincospi(2.0 * (double)j / (double)L, &s, &c);
    store_c(out, k, c, -s, dbl);
  }
}

// out[k] = exp(-pi*i*((a*k^2) mod L2)/(L2/2)), L2 = 2*d*N.
static __global__ void k_fill_chirp(void* out, int64_t count, uint64_t a, uint64_t L2, int dbl) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < count;
       k += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t kk = mulmod((uint64_t)k, (uint64_t)k, L2);
    const uint64_t j = mulmod(kk, a, L2);
    double s, c;
    sincospi(2.0 * (double)j / (double)L2, &s, &c);
    store_c(out, k, c, -s, dbl);
  }
}

// H[k] = (1/P) sum_j h[j] W_P^{jk}, h[j] = conj(chirp[j]) (j < M),
// conj(chirp[P-j]) (P-j < N), else 0.  Direct O(P^2) summation in FP64 with
// an exact W_P table (plan-time only).
static __global__ void k_chirp_kernel_fp64(double2* h, int P, int64_t n, int64_t m, uint64_t a, uint64_t L2) {
  // h[j] = conj(chirp[j]) (j < M), conj(chirp[P-j]) (P-j < N), else 0, in FP64
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < P; j += gridDim.x * blockDim.x) {
    int64_t src = -1;
    if (j < m)
      src = j;
    else if (P - j < n)
      src = P - j;
    double s = 0.0, c = 0.0;
    if (src >= 0) {
      const uint64_t jj = mulmod(mulmod((uint64_t)src, (uint64_t)src, L2), a, L2);
      sincospi(2.0 * (double)jj / (double)L2, &s, &c);
    }
    h[j] = make_double2(c, s);
  }
}

// H = FFT(h)/P at plan time: one radix-2 Stockham (autosort, decimation in
// frequency) level per launch in FP64 against the exact W_P table, ping-pong
// between two buffers; level `s` (stride, 1, 2, 4, ...) of sub-length ns = P/s:
// y[q + s 2p] = a + b, y[q + s (2p + 1)] = (a - b) W_ns^p with a = x[q + s p],
// b = x[q + s (p + ns/2)].  log2 P launches of P/2 butterflies replace the
// O(P^2) summation (2.4 ms at P = 16384).
static __global__ void k_stockham2_level(const double2* __restrict__ x, double2* __restrict__ y, int P, int s,
                                         const double2* __restrict__ wP) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P / 2) return;
  const int p = i / s, q = i - p * s, half = P / 2;
  const double2 a = x[q + s * p], b = x[q + s * p + half];
  const double2 w = __ldg(wP + p * s);
  const double dx = a.x - b.x, dy = a.y - b.y;
  y[q + s * 2 * p] = make_double2(a.x + b.x, a.y + b.y);
  y[q + s * (2 * p + 1)] = make_double2(dx * w.x - dy * w.y, dx * w.y + dy * w.x);
}

// out[k] = v[k] / P in the plan's element type
static __global__ void k_store_scaled(void* out, int P, const double2* __restrict__ v, int dbl) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < P) store_c(out, k, v[k].x / P, v[k].y / P, dbl);
}

// W[r, c] = W_L^{(a*r*c) mod L}, L = d*n, row-major rows x n.
static __global__ void k_dft_matrix(void* out, int64_t rows, int64_t n, uint64_t a, uint64_t L, int dbl) {
  const int64_t total = rows * n;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = i / n, c = i % n;
    const uint64_t j = mulmod(mulmod(a, r, L), c, L);
    double s, cc;
    sincospi(2.0 * (double)j / (double)L, &s, &cc);
    store_c(out, i, cc, -s, dbl);
  }
}

// ------------------------- reference building blocks -----------------------

template <typename Real>
static __global__ void k_combine(const void* y, const void* z, const void* tw, void* out, int64_t rows,
                          int64_t half) {
  using C = typename CT<Real>::T;
  const C* Y = reinterpret_cast<const C*>(y);
  const C* Z = reinterpret_cast<const C*>(z);
  const C* T = reinterpret_cast<const C*>(tw);
  C* O = reinterpret_cast<C*>(out);
  const int64_t total = rows * half;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / half, l = i % half;
    const C t = cmul(__ldg(T + l), __ldg(Z + i));
    const C yy = __ldg(Y + i);
    O[r * 2 * half + l] = cadd(yy, t);
    O[r * 2 * half + half + l] = csub(yy, t);
  }
}

template <typename Real>
static __global__ void k_block_sum(const void* x, void* out, int64_t rows, int64_t len) {
  using C = typename CT<Real>::T;
  const C* Xp = reinterpret_cast<const C*>(x);
  C* O = reinterpret_cast<C*>(out);
  const int64_t row = blockIdx.x;
  if (row >= rows) return;
  Real sx = 0, sy = 0;
  for (int64_t j = threadIdx.x; j < len; j += blockDim.x) {
    const C v = __ldg(Xp + row * len + j);
    sx += v.x;
    sy += v.y;
  }
  __shared__ Real red[2][32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sx += __shfl_down_sync(0xffffffffu, sx, o);
    sy += __shfl_down_sync(0xffffffffu, sy, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = sx;
    red[1][threadIdx.x >> 5] = sy;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    Real ax = 0, ay = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      ax += red[0][w];
      ay += red[1][w];
    }
    O[row] = mk(ax, ay);
  }
}

}  // namespace asx

// asx_afft_local.cuh — α-FFT for complex128 N = 4096 at α = 1/2 (reference
// DenseFactor(2), BASELINE config 1a) with group-local exchanges.
//
// The α-FFT splits the bins m = c + 2d into two output residues c ∈ {0, 1};
// residue c is the N-point DFT of x_n W_{2N}^{c n} (fastpath.py:162-181
// even/odd recursion restated per residue).  One CTA of two
// 256-thread teams transforms one signal at a time: team c computes residue
// c, both teams read the same TMA-staged input row.  Each 4096-point DFT is
// decimation in time over n = n0 + 16 n1 + 256 n2, d = g0 + 16 g1 + 256 g2:
//
//   S1  thread t = n0 + 16 n1 reads x[t + 256 n2] (the staged row, conflict-
//       free), × W_32^{c n2} (compile-time constants), radix-16 over n2 -> g0,
//       × W_{8192}^{t (c + 2 g0)} (exact, tensor memory)
//   E1  team-wide exchange (named barrier): -> thread (n0, g0)
//   S2  radix-16 over n1 -> g1, × W_256^{n0 g1} (exact, tensor memory)
//   E2  exchange inside the half-warp (__syncwarp): -> thread (g1, g0)
//   S3  radix-16 over n0 -> g2; only g2 < 8 (d < N/2, i.e. m < N) is kept
//   OUT both teams park their bins in their own half-warp regions; one signal
//       later (after the next signal's row reads and BEFORE its S1, behind a
//       split-phase "parked" mbarrier) all 512 threads write X[e] with e
//       contiguous across the warp (full 32-byte sectors: the residues
//       interleave as m = c + 2d); the stores drain during S1
//
// Per residue: one team-wide and one half-warp exchange (the Stockham engine
// needs three team-wide ones at R = 8), the α pre-twiddle folded into the
// S1 constants and the S1 twiddle table, and every FP64 operation is
// butterfly or twiddle work (no twiddle generation in the signal loop).  The
// per-thread twiddles come from a plan-time image (k_afl_image), copied into
// tensor memory once per CTA.
#pragma once

#include "asx_kernels.cuh"


namespace asx {

struct AfftLocal {
  static constexpr int P = 4096, TNT = 256, NTH = 512;
  static constexpr int RS = 272;        // region stride: 256 (E1) / 16 x 17 (E2) slots, conflict-free 16 B access
  static constexpr int XB = 16 * RS;    // one team's exchange buffer (complex128 elements)
  static constexpr size_t STAGE_OFF = size_t(2) * XB * sizeof(double2);
  static constexpr size_t ROW_BYTES = size_t(P) * sizeof(double2);
  static constexpr size_t BAR_OFF = STAGE_OFF + ROW_BYTES;
  static constexpr size_t SMEM = BAR_OFF + 5 * sizeof(uint64_t) + 16;  // full, consumed, war, -, parked, TMEM slot
  static constexpr int CPT = 128;       // TMEM columns per thread: S1 twiddles 16 x 4 | S2 twiddles 16 x 4
  static constexpr int IMG_ELEMS = 32 * NTH;  // twiddle image: [j < 32][thread < 512] complex128
  // parked output bin (g1, g2) of half-warp region hi of team c (conflict-free both ways)
  __host__ __device__ static constexpr int out_pos(int c, int hi, int g1, int g2) {
    return RS * hi + ((hi + 4 * c) & 7) + g1 + 16 * g2;
  }
};

// Plan-time image of every thread's tensor-memory twiddles (exact FP64
// sincospi of W_8192^k): img[j][tid], j < 16: W_8192^{t (c + 2 j)} (S1 of
// team c = tid / 256, t = tid % 256); j >= 16: W_256^{n0 (j - 16)}, n0 = t % 16.
static __global__ void k_afl_image(double2* img) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= AfftLocal::IMG_ELEMS) return;
  const int j = i / AfftLocal::NTH, tid = i % AfftLocal::NTH, c = tid / 256, t = tid % 256;
  const int k = j < 16 ? (t * (c + 2 * j)) & 8191 : (32 * (t & 15) * (j - 16)) & 8191;
  double sn, cs;
  sincospi(2.0 * double(k) / 8192.0, &sn, &cs);
  img[i] = make_double2(cs, -sn);
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}

// v[j] *= (twiddle j of this thread's 16-value TMEM block at column col), j >= J0
template <int J0>
__device__ __forceinline__ void afl_twiddle(double2 (&v)[16], uint32_t col) {
#pragma unroll
  for (int j0 = 0; j0 < 16; j0 += 4) {
    if (j0 + 3 < J0) continue;
    uint32_t w[16];
    tmem_ld16(col + 4 * j0, w);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (j0 + k >= J0) v[j0 + k] = cmul(v[j0 + k], words_to_c(&w[4 * k], (double2*)nullptr));
  }
}

// Timing diagnostics (variant builds only, -DASX_AFL_TIMELINE=<iteration>): warp
// leaders of CTA 0 stamp clock64() at the phase boundaries of two consecutive
// signals into the row AFTER the last output row (the caller allocates it).
#ifdef ASX_AFL_TIMELINE
#define AFL_TL(i)                                                                                   \
  do {                                                                                              \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && (it == ASX_AFL_TIMELINE || it == ASX_AFL_TIMELINE + 1)) \
      cx.tl[((it - ASX_AFL_TIMELINE) * 16 + (threadIdx.x >> 5)) * 16 + (i)] = clock64();           \
  } while (0)
#else
#define AFL_TL(i)
#endif

struct AflCtx {
  unsigned long long* tl;
  double2* xb;  // this team's exchange buffer
  const unsigned char* stage;
  uint64_t *full, *consumed, *war;
  uint32_t tbase;
  int t;
  double2* xb0;      // both teams' buffers (the parked bins)
  uint64_t* parked;  // every warp has parked its bins
};

// X[e], e = c + 2d for the parked bins of signal u: contiguous across the
// warp (full 32-byte sectors; residue c = e & 1 comes from team c's buffer)
__device__ __forceinline__ void afl_copyout(const KParams& p, const double2* xb0, int u, int tid) {
  using L = AfftLocal;
  using C = double2;
  C* X = reinterpret_cast<C*>(p.X) + int64_t(u) * p.Xs;
  const bool full_row = p.m >= L::P;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int e = tid + L::NTH * j, c = e & 1, d = e >> 1;
    const C val = xb0[c * L::XB + L::out_pos(c, d & 15, (d >> 4) & 15, d >> 8)];
    if (full_row || e < p.m) X[e] = val;
  }
}

// One signal's residue CR on this team (t = team-local thread), up to the
// parked outputs.
template <int CR>
__device__ __forceinline__ void afl_residue(const KParams& p, const AflCtx& cx, int u, int it, int stride,
                                            bool live, uint32_t& phase, uint32_t xcnt, bool live_prev) {
  using L = AfftLocal;
  using C = double2;
  const int t = cx.t, n0 = t & 15, hi = t >> 4;
  C v[16];
  AFL_TL(0);
  if (live) {
    mbar_wait(cx.full, phase);
    phase ^= 1;
    AFL_TL(1);
    const C* row = reinterpret_cast<const C*>(cx.stage);
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = row[t + 256 * i];
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = mk(0.0, 0.0);
  }
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(cx.consumed);  // this warp is done with the staged row
  AFL_TL(2);
  if (xcnt) {
    // The previous signal's bins, parked by both teams at the end of the last
    // iteration: write them now, BEFORE this signal's butterflies.  The 64 KiB
    // of global stores drain through the SM's 32 B/clk store path in ~2 k
    // cycles; issued here they drain while S1 keeps the FP64 pipe busy, issued
    // after S1 (round 1) they sat in the LSU queue in front of the E1
    // shared-memory stores (0.1517 -> 0.1409 ms, profiles/r2_c1a_experiments.md).
    mbar_wait(cx.parked, (xcnt - 1) & 1);
    if (live_prev) afl_copyout(p, cx.xb0, u - stride, threadIdx.x);
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(cx.war);
  }
  // ---- S1: × W_32^{c n2}, radix-16 over n2, × W_8192^{t (c + 2 g0)}
  if constexpr (CR == 1) {
#pragma unroll
    for (int i = 1; i < 16; ++i) v[i] = tw_const<32>(v[i], i);
  }
  ASX_DFT16_F64(v);
  afl_twiddle<CR == 0 ? 1 : 0>(v, cx.tbase);
  AFL_TL(3);
  AFL_TL(4);
  // ---- E1: (t, g0) -> thread (n0, g0); WAR: the previous signal's output reads
  if (xcnt) mbar_wait(cx.war, (xcnt - 1) & 1);
  AFL_TL(5);
  C* const xb = cx.xb;
#pragma unroll
  for (int g0 = 0; g0 < 16; ++g0) xb[t + L::RS * g0] = v[g0];
  AFL_TL(6);
  asm volatile("bar.sync %0, 256;" ::"r"(1 + CR) : "memory");
  AFL_TL(7);
  if (CR == 0 && t == 0 && u + stride < int(p.batch)) {
    // next row: both teams started this signal together and have read it by now
    mbar_wait(cx.consumed, it & 1);
    fence_proxy_async();
    mbar_expect_tx(cx.full, (uint32_t)L::ROW_BYTES);
    tma_load_1d(const_cast<unsigned char*>(cx.stage),
                static_cast<const unsigned char*>(p.x) + int64_t(u + stride) * p.xs * int64_t(sizeof(C)),
                (uint32_t)L::ROW_BYTES, cx.full);
  }
  C* rg = xb + L::RS * hi;  // this half-warp's region (g0 = hi)
#pragma unroll
  for (int n1 = 0; n1 < 16; ++n1) v[n1] = rg[n0 + 16 * n1];
  __syncwarp();
  AFL_TL(8);
  // ---- S2: radix-16 over n1, × W_256^{n0 g1}
  ASX_DFT16_F64(v);
  afl_twiddle<1>(v, cx.tbase + 64);
  AFL_TL(9);
  // ---- E2 (half-warp): (n0, g1) -> thread (g1 = t & 15, g0)
#pragma unroll
  for (int g1 = 0; g1 < 16; ++g1) rg[n0 + 17 * g1] = v[g1];
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = rg[j + 17 * n0];
  __syncwarp();
  AFL_TL(10);
  // ---- S3: radix-16 over n0 -> g2; park bins d = hi + 16 n0 + 256 g2 < 2048
  ASX_DFT16_F64(v);
  AFL_TL(11);
#pragma unroll
  for (int g2 = 0; g2 < 8; ++g2) xb[L::out_pos(CR, hi, n0, g2)] = v[g2];
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(cx.parked);
  AFL_TL(12);
}

// Launch: grid <= #SMs, NTH threads, AfftLocal::SMEM dynamic shared memory.
// Preconditions (host): complex128 input, n = 4096, r = 2, fold = 1,
// m <= 4096, 16-byte aligned rows, batch < 2^31, p.afl = the plan's image.
template <typename Real>
__global__ void __launch_bounds__(512, 1) k_afft_local(KParams p) {
  static_assert(sizeof(Real) == 8, "complex128 kernel");
  using L = AfftLocal;
  using C = double2;
  extern __shared__ __align__(128) unsigned char smraw[];
  const int tid = threadIdx.x, team = tid >> 8, warp = tid >> 5;
  C* const xb0 = reinterpret_cast<C*>(smraw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smraw + L::BAR_OFF);
  uint32_t& tmem_slot = *reinterpret_cast<uint32_t*>(bars + 5);
  AflCtx cx;
  cx.xb = xb0 + team * L::XB;
  cx.stage = smraw + L::STAGE_OFF;
  cx.full = bars;
  cx.consumed = bars + 1;
  cx.war = bars + 2;
  cx.parked = bars + 4;
  cx.xb0 = xb0;
  cx.t = tid & 255;
  cx.tl = reinterpret_cast<unsigned long long*>(reinterpret_cast<C*>(p.X) + int64_t(p.batch) * p.Xs);
  const int stride = int(gridDim.x);
  int u = int(blockIdx.x);
  const int batch = int(p.batch);
  const int iters = (batch + stride - 1) / stride;
  if (tid == 0) {
    mbar_init(cx.full, 1);
    mbar_init(cx.consumed, L::NTH / 32);
    mbar_init(cx.war, L::NTH / 32);
    mbar_init(cx.parked, L::NTH / 32);
    fence_mbar_init();
    if (u < batch) {  // first row in flight while the twiddles go to tensor memory
      mbar_expect_tx(cx.full, (uint32_t)L::ROW_BYTES);
      tma_load_1d(const_cast<unsigned char*>(cx.stage),
                  static_cast<const unsigned char*>(p.x) + int64_t(u) * p.xs * int64_t(sizeof(C)),
                  (uint32_t)L::ROW_BYTES, cx.full);
    }
  }
  if (warp == 0) tmem_alloc(&tmem_slot, 512);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  cx.tbase = tmem_slot + (uint32_t(32 * (warp & 3)) << 16) + uint32_t((warp >> 2) * L::CPT);
  {
    const double2* img = reinterpret_cast<const double2*>(p.afl) + tid;
#pragma unroll 1
    for (int j0 = 0; j0 < 32; j0 += 16) {
      double2 w[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) w[j] = __ldg(img + L::NTH * (j0 + j));
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        uint32_t w8[8];
        c_to_words(w[j], &w8[0]);
        c_to_words(w[j + 1], &w8[4]);
        tmem_st8(cx.tbase + 4 * (j0 + j), w8);
      }
    }
    tmem_wait_st();
  }
  __syncthreads();
  uint32_t phase = 0, xcnt = 0;
#pragma unroll 1
  for (int it = 0; it < iters; ++it, u += stride) {
    const bool live = u < batch;
    const bool live_prev = u - stride < batch;
    if (team == 0)
      afl_residue<0>(p, cx, u, it, stride, live, phase, xcnt, live_prev);
    else
      afl_residue<1>(p, cx, u, it, stride, live, phase, xcnt, live_prev);
    ++xcnt;
  }
  if (xcnt) {  // the last signal's bins
    const int u_last = u - stride;
    mbar_wait(cx.parked, (xcnt - 1) & 1);
    if (u_last < batch) afl_copyout(p, xb0, u_last, tid);
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 0) tmem_dealloc(tmem_slot, 512);
}

}  // namespace asx

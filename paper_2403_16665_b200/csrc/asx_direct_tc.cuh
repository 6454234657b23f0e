// asx_direct_tc.cuh — direct α-DFT of complex64 signals on the 5th-generation
// tensor cores (tcgen05.mma kind::f16, accumulators in tensor memory).
//
// The direct form (oracle.py:37-67 `_reduced_product` / `naive_forward`,
// batched as the reference's acceptance test does, test_acceptance.py:64-67)
// is the contraction X[b, m] = Σ_n x[b, n]·W[m, n].  Read as reals it is one
// GEMM with no reshuffling of the data:
//
//     C[b, j] = Σ_k A[b, k] · V[j, k]       A = x as float[B][2N] (re, im interleaved)
//                                             C = X as float[B][2M]
//     V[2m,   2n] =  Re W   V[2m,   2n+1] = -Im W
//     V[2m+1, 2n] =  Im W   V[2m+1, 2n+1] =  Re W
//
// complex64 needs ~fp32 products (tolerance 2e-5 of max|X|).  Each operand is
// split into two fp16 terms, v = hi + lo, hi = fp16(v), lo = fp16(v - hi),
// and C = A_hi·V_hi + A_hi·V_lo + A_lo·V_hi with fp32 accumulation (the
// dropped lo·lo term is ~2^-22 relative).  To keep the fp16 terms in range for
// any input, every signal is scaled by a power of two so that its max |x|
// lands in [2^10, 2^11), V by 2^8; the epilogue multiplies the exact inverse.
//
// One persistent CTA per SM, 128 signals per tile (= MMA M = the 128 TMEM
// lanes), all 2M <= 512 output reals of the tile accumulated in TMEM (N = 256
// per MMA, M <= 256 bins).  K streams in chunks of 64 reals (one 128-byte
// swizzled fp16 row per operand row):
//   warps 0-7   convert: x (fp32, coalesced float4 loads) -> scaled fp16 hi/lo
//               in the SWIZZLE_128B K-major layout, 2-stage ring; then the
//               epilogue of the previous tile (tcgen05.ld -> scale -> store)
//   warp 8      one elected thread issues the MMAs (3 per 16-wide K step)
//   warp 9      one thread streams V's plan-time fp16 image (already swizzled)
//               by 1-D TMA bulk copies, 2-stage ring of 64 KB stages
//   warps 10-13 per-signal scales of the next tile (first, HBM-bound read of x)
// ---------------------------------------------------------------------------
#pragma once

#include <cuda_fp16.h>

#include "asx_engine.cuh"

namespace asx {
namespace dtc {

constexpr int TS = 128;                   // signals per tile
constexpr int KC = 64;                    // reals per K chunk
constexpr int NMMA = 256;                 // output reals per MMA
constexpr int NCONV = 256;                // converter / epilogue threads
constexpr int NSCALE = 128;               // row-scale warps (one tile ahead; their reads warm L2)
constexpr int NTHREADS = NCONV + 64 + NSCALE;  // + MMA warp + V-loader warp + scale warps
constexpr int A_HALF = TS * KC * 2;       // one fp16 term of an A stage: 16 KB
constexpr int A_STAGE = 2 * A_HALF;       // hi + lo
constexpr int B_HALF = NMMA * KC * 2;     // 32 KB
constexpr int B_STAGE = 2 * B_HALF;       // hi + lo: 64 KB
constexpr int NA = 2, NB = 2;
constexpr float V_SCALE = 256.0f;
constexpr int SMEM_BYTES = 1024 /*align*/ + NA * A_STAGE + NB * B_STAGE + 1024 /*bars, slot*/ + 2 * TS * 4 /*scales*/;
constexpr int TMEM_COLS = 512;

struct Params {
  const float* x;   // float view of complex64 input
  int64_t xs;       // row stride, complex elements
  float* X;
  int64_t Xs;       // output row stride, complex elements
  int64_t batch;
  int n, m;         // complex length / bins; 2n % 64 == 0, m % 128 == 0, m <= 256
  const unsigned char* vimg;  // plan-time image: [kc][half][hi|lo][256][64] fp16, swizzled
};

// byte offset of element (row, k) of a K-major SWIZZLE_128B tile of 64-wide fp16 rows
__host__ __device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t k) {
  return row * 128u + ((((k >> 3) ^ (row & 7u)) & 7u) << 4) + (k & 7u) * 2u;
}

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4)  // start address
         | ((uint64_t)1 << 16)                 // LBO (unused for swizzled K-major)
         | ((uint64_t)(1024 >> 4) << 32)       // SBO: 8 rows x 128 B
         | ((uint64_t)1 << 46)                 // sm_100 descriptor version
         | ((uint64_t)2 << 61);                // SWIZZLE_128B
}
// kind::f16: fp16 x fp16 -> fp32, both K-major, M = 128, N = 256
constexpr uint32_t IDESC = (1u << 4) | (uint32_t(NMMA >> 3) << 17) | (uint32_t(TS >> 4) << 24);

__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(IDESC), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}

__device__ __forceinline__ uint32_t pack_h2(__half a, __half b) {
  return (uint32_t)__half_as_ushort(a) | ((uint32_t)__half_as_ushort(b) << 16);
}
__device__ __forceinline__ void split4(float4 v, float s, uint2& hi, uint2& lo) {
  const float f[4] = {v.x * s, v.y * s, v.z * s, v.w * s};
  __half h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    h[i] = __float2half_rn(f[i]);
    l[i] = __float2half_rn(f[i] - __half2float(h[i]));
  }
  hi = make_uint2(pack_h2(h[0], h[1]), pack_h2(h[2], h[3]));
  lo = make_uint2(pack_h2(l[0], l[1]), pack_h2(l[2], l[3]));
}

__global__ void __launch_bounds__(NTHREADS, 1) k_direct_tc(Params p) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sA = smem;                       // NA x [hi 16 KB | lo 16 KB]
  unsigned char* sB = smem + NA * A_STAGE;        // NB x [hi 32 KB | lo 32 KB]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + NB * B_STAGE);
  uint64_t* a_full = bars;           // NA, count NCONV
  uint64_t* a_empty = bars + NA;     // NA, tcgen05.commit
  uint64_t* b_full = bars + 2 * NA;  // NB, TMA tx
  uint64_t* b_empty = b_full + NB;   // NB, tcgen05.commit
  uint64_t* acc_full = b_empty + NB; // tcgen05.commit
  uint64_t* acc_empty = acc_full + 1;  // count NCONV
  uint64_t* sc_full = acc_empty + 1;   // 2, count NSCALE
  uint64_t* sc_empty = sc_full + 2;    // 2, count NCONV
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sc_empty + 2);
  float* scale = reinterpret_cast<float*>(smem + NA * A_STAGE + NB * B_STAGE + 1024);  // [2][TS]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kcn = (2 * p.n) / KC;       // K chunks
  const int nh = (2 * p.m) / NMMA;      // MMAs per K step (output halves)
  const int64_t ntiles = (p.batch + TS - 1) / TS;

  if (tid == 0) {
    for (int i = 0; i < NA; ++i) {
      mbar_init(&a_full[i], NCONV);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < NB; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, NCONV);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sc_full[i], NSCALE);
      mbar_init(&sc_empty[i], NCONV);
    }
    fence_mbar_init();
  }
  if (warp == 8) tmem_alloc(tmem_slot, TMEM_COLS);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 8) {
    // ------------------------------ converters + epilogue ------------------------------
    uint32_t ca = 0;  // A chunks produced
    int64_t prev = -1;
    uint32_t ntile_done = 0;
    auto convert = [&](int64_t t, int buf, int c) {
      const uint32_t s = ca % NA;
      float4 v[8];
      const float* sc = scale + buf * TS;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int q = tid + NCONV * i, row = q >> 4, c4 = q & 15;
        const int64_t b = t * TS + row;
        v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (b < p.batch)
          v[i] = __ldg(reinterpret_cast<const float4*>(p.x + b * 2 * p.xs + c * KC + c4 * 4));
      }
      mbar_wait(&a_empty[s], ((ca / NA) & 1) ^ 1);
      unsigned char* st = sA + s * A_STAGE;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int q = tid + NCONV * i, row = q >> 4, c4 = q & 15;
        uint2 hi, lo;
        split4(v[i], sc[row], hi, lo);
        const uint32_t off = swz(row, c4 * 4);
        *reinterpret_cast<uint2*>(st + off) = hi;
        *reinterpret_cast<uint2*>(st + A_HALF + off) = lo;
      }
      fence_proxy_async();
      mbar_arrive(&a_full[s]);
      ++ca;
    };
    auto epilogue = [&](int64_t t, int buf) {
      mbar_wait(acc_full, ntile_done & 1);
      tmem_fence_after();
      const int q = warp & 3, h = warp >> 2;
      const int r = q * 32 + lane;
      const int64_t b = t * TS + r;
      const float inv = 1.f / (scale[buf * TS + r] * V_SCALE);
      const int cols = p.m;  // output reals per warp group (2m split in two)
      for (int c0 = 0; c0 < cols; c0 += 32) {
        uint32_t w[32];
        const int col = h * cols + c0;
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)col, w);
        if (b < p.batch) {
          float4* dst = reinterpret_cast<float4*>(p.X + b * 2 * p.Xs + col);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            dst[i] = make_float4(__uint_as_float(w[4 * i]) * inv, __uint_as_float(w[4 * i + 1]) * inv,
                                 __uint_as_float(w[4 * i + 2]) * inv, __uint_as_float(w[4 * i + 3]) * inv);
        }
      }
      tmem_fence_before();
      mbar_arrive(acc_empty);
      mbar_arrive(&sc_empty[buf]);
      ++ntile_done;
    };
    int it = 0;  // tiles of this CTA so far; scale buffer = it & 1
    for (int64_t t = blockIdx.x;; t += gridDim.x, ++it) {
      const bool valid = t < ntiles;
      if (valid) {
        mbar_wait(&sc_full[it & 1], (it >> 1) & 1);
        for (int c = 0; c < NA && c < kcn; ++c) convert(t, it & 1, c);
      }
      if (prev >= 0) epilogue(prev, (it - 1) & 1);
      if (!valid) break;
      for (int c = NA; c < kcn; ++c) convert(t, it & 1, c);
      prev = t;
    }
  } else if (warp == 8) {
    // ------------------------------ MMA issuer ------------------------------
    if (lane == 0) {
      uint32_t ca = 0, cb = 0, nt = 0;
      const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++nt) {
        if (nt > 0) {
          mbar_wait(acc_empty, (nt - 1) & 1);
          tmem_fence_after();
        }
        for (int c = 0; c < kcn; ++c) {
          const uint32_t sa = ca % NA;
          mbar_wait(&a_full[sa], (ca / NA) & 1);
          tmem_fence_after();
          const uint32_t ah = a0 + sa * A_STAGE, al = ah + A_HALF;
          for (int hh = 0; hh < nh; ++hh) {
            const uint32_t sb = cb % NB;
            mbar_wait(&b_full[sb], (cb / NB) & 1);
            tmem_fence_after();
            const uint32_t bh = b0 + sb * B_STAGE, bl = bh + B_HALF;
            const uint32_t d = tmem + (uint32_t)(hh * NMMA);
#pragma unroll
            for (int k = 0; k < KC / 16; ++k) {
              const uint32_t ko = k * 32;  // 16 fp16 = 32 bytes along the swizzled row
              mma_f16(d, sdesc(ah + ko), sdesc(bh + ko), (c > 0 || k > 0) ? 1u : 0u);
              mma_f16(d, sdesc(ah + ko), sdesc(bl + ko), 1u);
              mma_f16(d, sdesc(al + ko), sdesc(bh + ko), 1u);
            }
            mma_commit(&b_empty[sb]);
            ++cb;
          }
          mma_commit(&a_empty[sa]);
          ++ca;
        }
        mma_commit(acc_full);
      }
    }
    __syncwarp();
  } else if (warp >= 10) {
    // ---------------- row scales, one tile ahead of the converters ----------------
    // Power of two per signal so its max |x| lands in [2^10, 2^11).  Each warp
    // takes 32 rows, four at a time with all their loads in flight; the reads
    // also bring the tile into L2 for the converters.
    const int sw = warp - 10;
    int it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int buf = it & 1;
      mbar_wait(&sc_empty[buf], ((it >> 1) & 1) ^ 1);
      float* sc = scale + buf * TS;
      for (int r0 = sw * 32; r0 < sw * 32 + 32; r0 += 4) {
        float mx[4] = {0.f, 0.f, 0.f, 0.f};
        const int nq = p.n / 2;  // float4 per row
        for (int i0 = 0; i0 < nq; i0 += 128) {
          float4 v[4][4];
#pragma unroll
          for (int rr = 0; rr < 4; ++rr) {
            const int64_t b = t * TS + r0 + rr;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int i = i0 + lane + 32 * u;
              v[rr][u] = make_float4(0.f, 0.f, 0.f, 0.f);
              if (b < p.batch && i < nq) v[rr][u] = __ldg(reinterpret_cast<const float4*>(p.x + b * 2 * p.xs) + i);
            }
          }
#pragma unroll
          for (int rr = 0; rr < 4; ++rr)
#pragma unroll
            for (int u = 0; u < 4; ++u)
              mx[rr] = fmaxf(mx[rr], fmaxf(fmaxf(fabsf(v[rr][u].x), fabsf(v[rr][u].y)),
                                           fmaxf(fabsf(v[rr][u].z), fabsf(v[rr][u].w))));
        }
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) mx[rr] = fmaxf(mx[rr], __shfl_xor_sync(0xffffffffu, mx[rr], o));
          if (lane == rr) {
            float sv = 1.f;
            if (mx[rr] > 0.f && mx[rr] <= 3.0e38f) sv = exp2f((float)(10 - ilogbf(mx[rr])));
            sc[r0 + rr] = sv;
          }
        }
      }
      mbar_arrive(&sc_full[buf]);
    }
  } else {
    // ------------------------------ V image loader ------------------------------
    if (lane == 0) {
      uint32_t cb = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int c = 0; c < kcn; ++c) {
          for (int hh = 0; hh < nh; ++hh) {
            const uint32_t sb = cb % NB;
            mbar_wait(&b_empty[sb], ((cb / NB) & 1) ^ 1);
            mbar_expect_tx(&b_full[sb], B_STAGE);
            const unsigned char* src = p.vimg + (size_t)(c * nh + hh) * B_STAGE;
            unsigned char* dst = sB + sb * B_STAGE;
#pragma unroll
            for (int i = 0; i < 4; ++i) tma_load_1d(dst + i * (B_STAGE / 4), src + i * (B_STAGE / 4), B_STAGE / 4, &b_full[sb]);
            ++cb;
          }
        }
      }
    }
    __syncwarp();
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 8) tmem_dealloc(tmem, TMEM_COLS);
}

// Plan time: the real-ified, scaled, fp16-split V image in the shared-memory
// layout the MMA reads (so the loader is a plain bulk copy).  Phases use the
// exact integer reduction (a·m·n) mod L of oracle.py:37-47 and sincospi.
__global__ void k_direct_tc_image(unsigned char* img, int n, int m, uint64_t a, uint64_t L) {
  const int nh = (2 * m) / NMMA;
  const int64_t total = (int64_t)(2 * n) * (2 * m);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e / (2 * n)), kk = (int)(e % (2 * n));  // output real j, input real kk
    const int mb = j >> 1, nn = kk >> 1;
    const uint64_t ph = (uint64_t)(((unsigned __int128)((uint64_t)a * (uint64_t)mb) * (uint64_t)nn) % L);
    double sn, cs;
    sincospi(2.0 * (double)ph / (double)L, &sn, &cs);  // W = cs - i sn
    const double wr = cs, wi = -sn;
    double v;
    if ((j & 1) == 0)
      v = (kk & 1) == 0 ? wr : -wi;
    else
      v = (kk & 1) == 0 ? wi : wr;
    v *= (double)V_SCALE;
    const __half hi = __float2half_rn((float)v);
    const __half lo = __float2half_rn((float)(v - (double)__half2float(hi)));
    const int c = kk / KC, k = kk % KC, hh = j / NMMA, row = j % NMMA;
    unsigned char* st = img + (size_t)(c * nh + hh) * B_STAGE;
    const uint32_t off = swz((uint32_t)row, (uint32_t)k);
    *reinterpret_cast<__half*>(st + off) = hi;
    *reinterpret_cast<__half*>(st + B_HALF + off) = lo;
  }
}

}  // namespace dtc
}  // namespace asx

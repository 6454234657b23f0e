// asx_direct_tc2.cuh — the tensor-core direct α-DFT on CTA pairs
// (tcgen05.mma.cta_group::2), for complex64 plans with M = 256 bins
// (BASELINE config 3).
//
// Same arithmetic as k_direct_tc (asx_direct_tc.cuh: fp16 hi/lo splits,
// three products per real GEMM, fp32 accumulation in tensor memory,
// per-signal power-of-two scaling), with the roles of the operands swapped
// so the accumulator of a tile fits in HALF of each SM's tensor memory:
//
//   D[bin][signal] = Σ_k W[bin][k] · x[signal][k]        (MMA M = 256 bins,
//                                                        N = 128 signals)
//
// On a CTA pair the M = 256 rows are split across the two SMs (CTA r holds W
// rows = bins 128r..128r+127 in its shared memory and D rows 128r.. in its
// tensor memory) and the N = 128 columns of B across their shared memories
// (CTA r converts signals 64r..64r+63 of the tile), cute's 2x1SM layouts
// (mma_traits_sm100.hpp SM100_MMA_F16BF16_2x1SM_SS).  Re and Im of a tile take
// 2 x 128 columns per SM, so two accumulator buffers fit in the 512 columns
// and the epilogue of tile t drains while the MMAs of tile t+1 run -- the
// serialisation that bounds k_direct_tc.  Per SM and MMA the
// shared-memory operand reads are its 128 W rows and 64 x rows.
//
// Warp roles (both CTAs; only rank 0 issues MMAs):
//   0-7    converters: x (fp32, coalesced) -> scaled fp16 hi/lo terms of the
//          CTA's 64 signals, K-major SWIZZLE_64B B stages
//   8-11   epilogue: tcgen05.ld 32x32b (lane = bin, column = signal) ->
//          × exact inverse scale -> 256-byte row segments of X per store
//   12     MMA issuer (rank 0, one thread): 24 MMAs of 256x128x16 per
//          32-sample chunk
//   13     W loader: the CTA's 32 KB half of the W chunk by one bulk copy
//   14     W relay: re-arms rank 0's "W ready" barrier once this CTA's half
//          has landed (a bulk copy completes on a barrier of its own CTA)
//   15-22  per-signal scales of the CTA's 64 signals, one tile ahead,
//          written to both CTAs' shared memory (the epilogue of each CTA
//          scales all 128 signals of the tile)
#pragma once

#include <cuda_fp16.h>

#include "asx_direct_tc.cuh"

#ifndef ASX_DTC2_ABLATE
#define ASX_DTC2_ABLATE 0  // timing-only ablation builds (`make variant`, wrong results): 1 no MMAs, 2 no
                           // epilogue stores, 4 no x loads in the converters, 8 no scale pass loads, 16 no W
                           // bulk copies.  0 shipped.
#endif

namespace asx {
namespace dtc2 {

constexpr int TS = 128;                  // signals per pair tile (MMA N)
constexpr int HS = 64;                   // signals per CTA
constexpr int MB = 256;                  // bins (MMA M, 128 per CTA)
constexpr int KC = 32;                   // samples per chunk
constexpr int NCONV = 256, NEPI = 128, NSCALE = 256;
constexpr int WR_CONV = 0, WR_EPI = 8, WR_MMA = 12, WR_LOAD = 13, WR_RELAY = 14, WR_SCALE = 15;
constexpr int NTHREADS = 32 * 23;
constexpr int X_TERM = HS * KC * 2;      // one fp16 term of 64 signals: 4 KB
constexpr int X_STAGE = 4 * X_TERM;      // [xr hi | xr lo | xi hi | xi lo]
constexpr int W_TERM = 128 * KC * 2;     // one fp16 term of 128 bins: 8 KB
constexpr int W_STAGE = 4 * W_TERM;      // [Wr hi | Wr lo | Wi hi | Wi lo]
#ifndef ASX_DTC2_NX
#define ASX_DTC2_NX 4
#endif
#ifndef ASX_DTC2_NW
#define ASX_DTC2_NW 3
#endif
constexpr int NX = ASX_DTC2_NX, NW = ASX_DTC2_NW, NSC = 3;
constexpr int ACC_COLS = 2 * TS;         // Re | Im of one tile
constexpr float W_SCALE = 256.0f;
constexpr int SCALE_BYTES = NSC * TS * 16;  // float4 (f1, f2, 1/f1, 1/(f2 W_SCALE)) per signal
constexpr int SMEM_BYTES = 1024 + NW * W_STAGE + NX * X_STAGE + SCALE_BYTES + 512;

struct Params {
  const float* x;
  int64_t xs;
  float* X;
  int64_t Xs;
  int64_t batch;
  int n;                      // n % 32 == 0, n <= 1024; m == 256
  const unsigned char* wimg;  // [chunk][cta][Wr hi | Wr lo | Wi hi | Wi lo][128][32] fp16, swizzled
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of a local shared-memory object in CTA `rank`
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// release at cluster scope: for data the peer reads with generic loads (the
// scales); costs a GPU-scope membar, so only once per tile
__device__ __forceinline__ void arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// plain remote arrive (default semantics): hand-offs whose data is read by the
// tensor core's async proxy (after fence.proxy.async) or lives in tensor memory
__device__ __forceinline__ void arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ bool try_wait_cluster(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void wait_cluster(uint64_t* bar, uint32_t phase) {
  while (!try_wait_cluster(bar, phase)) {
  }
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void st_cluster_f4(uint32_t cluster_addr, float4 v) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(cluster_addr), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void mma2_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
// completion of every MMA issued so far -> the barrier at this offset in BOTH CTAs
__device__ __forceinline__ void commit2(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
// kind::f16, fp32 D, both K-major, M = 256 (pair), N = 128
__device__ __forceinline__ uint32_t idesc2(bool neg_a) {
  return (1u << 4) | (neg_a ? (1u << 13) : 0u) | (uint32_t(TS >> 3) << 17) | (uint32_t(MB >> 4) << 24);
}
// Re and Im columns of one 16-signal block, wait fused: the registers cannot
// be consumed before the loads have landed
__device__ __forceinline__ void tmem_ld_re_im(uint32_t a_re, uint32_t a_im, uint32_t (&re)[16], uint32_t (&im)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%32];\n"
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%33];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(re[0]), "=r"(re[1]), "=r"(re[2]), "=r"(re[3]), "=r"(re[4]), "=r"(re[5]), "=r"(re[6]), "=r"(re[7]), "=r"(re[8]), "=r"(re[9]), "=r"(re[10]), "=r"(re[11]), "=r"(re[12]), "=r"(re[13]), "=r"(re[14]), "=r"(re[15]), "=r"(im[0]), "=r"(im[1]), "=r"(im[2]), "=r"(im[3]), "=r"(im[4]), "=r"(im[5]), "=r"(im[6]), "=r"(im[7]), "=r"(im[8]), "=r"(im[9]), "=r"(im[10]), "=r"(im[11]), "=r"(im[12]), "=r"(im[13]), "=r"(im[14]), "=r"(im[15])
      : "r"(a_re), "r"(a_im)
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS, 1) k_direct_tc2(Params p) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sW = smem;                    // NW x W_STAGE
  unsigned char* sX = sW + NW * W_STAGE;       // NX x X_STAGE
  float4* scale = reinterpret_cast<float4*>(sX + NX * X_STAGE);  // [NSC][TS]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sX + NX * X_STAGE + SCALE_BYTES);
  uint64_t* w_full = bars;                // NW  local TMA
  uint64_t* w_ready = w_full + NW;        // NW  rank 0: one relay arrival per CTA
  uint64_t* w_empty = w_ready + NW;       // NW  MMA commit (multicast)
  uint64_t* x_full = w_empty + NW;        // NX  rank 0: converter warps of both CTAs
  uint64_t* x_empty = x_full + NX;        // NX  MMA commit (multicast)
  uint64_t* acc_full = x_empty + NX;      // 2   MMA commit (multicast)
  uint64_t* acc_empty = acc_full + 2;     // 2   rank 0: epilogue warps of both CTAs
  uint64_t* sc_full = acc_empty + 2;      // NSC scale warps of both CTAs
  uint64_t* sc_empty = sc_full + NSC;     // NSC local converters + epilogues of both CTAs
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sc_empty + NSC);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_rank(), peer = rank ^ 1u;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int kcn = p.n / KC;
  const int64_t ntiles = (p.batch + TS - 1) / TS;

  if (tid == 0) {
    for (int i = 0; i < NW; ++i) {
      mbar_init(&w_full[i], 1);
      mbar_init(&w_ready[i], 2);
      mbar_init(&w_empty[i], 1);
    }
    for (int i = 0; i < NX; ++i) {
      mbar_init(&x_full[i], 2 * (NCONV / 32));
      mbar_init(&x_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 2 * (NEPI / 32));
    }
    for (int i = 0; i < NSC; ++i) {
      mbar_init(&sc_full[i], 2 * (NSCALE / 32));
      mbar_init(&sc_empty[i], NCONV / 32 + 2 * (NEPI / 32));
    }
    fence_mbar_init();
  }
  if (warp == WR_MMA) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tmem_fence_before();
  cluster_sync();  // barriers and TMEM of both CTAs exist before any remote access
  tmem_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < WR_EPI) {
    // ------------------------------ converters ------------------------------
    // 64 rows x 32 complex (256 B) of x per chunk; a thread takes 4 consecutive
    // complex, twice.  The next chunk's loads (of this tile or the next) are in
    // flight while the current one is converted.
    uint32_t cx = 0;  // x chunks produced
    const uint32_t xfull0 = mapa(smem_u32(x_full), 0);
    auto load = [&](int64_t t, int c, float4 (&v)[2][2]) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int q = tid + NCONV * i, row = q >> 3, g = q & 7;
        const int64_t b = t * TS + HS * rank + row;
        v[i][0] = v[i][1] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (b < p.batch && !(ASX_DTC2_ABLATE & 4)) {
          const float4* src = reinterpret_cast<const float4*>(p.x + b * 2 * p.xs + (int64_t)c * 2 * KC) + 2 * g;
          v[i][0] = __ldcs(src);
          v[i][1] = __ldcs(src + 1);
        }
      }
    };
    float4 v[2][2], vn[2][2];
    int64_t t = pair;
    int c = 0, it = 0;
    if (t < ntiles) load(t, 0, v);
    while (t < ntiles) {
      int64_t tn = t;
      int cn = c + 1;
      if (cn == kcn) {
        cn = 0;
        tn += npairs;
      }
      if (tn < ntiles) load(tn, cn, vn);
      const int sb = it % NSC;
      if (c == 0) wait_cluster(&sc_full[sb], (it / NSC) & 1);
      const float4* sc = scale + sb * TS + HS * rank;
      const uint32_t s = cx % NX;
      mbar_wait(&x_empty[s], ((cx / NX) & 1) ^ 1);
      unsigned char* st = sX + s * X_STAGE;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int q = tid + NCONV * i, row = q >> 3, g = q & 7;
        const float4 f = sc[row];
        const float a = f.x, bb = f.y;
        uint2 rh, rl, ih, il;
        dtc::split2(v[i][0].x * a * bb, v[i][0].z * a * bb, rh.x, rl.x);
        dtc::split2(v[i][1].x * a * bb, v[i][1].z * a * bb, rh.y, rl.y);
        dtc::split2(v[i][0].y * a * bb, v[i][0].w * a * bb, ih.x, il.x);
        dtc::split2(v[i][1].y * a * bb, v[i][1].w * a * bb, ih.y, il.y);
        const uint32_t off = dtc::swz(row, 4 * g);
        *reinterpret_cast<uint2*>(st + off) = rh;
        *reinterpret_cast<uint2*>(st + X_TERM + off) = rl;
        *reinterpret_cast<uint2*>(st + 2 * X_TERM + off) = ih;
        *reinterpret_cast<uint2*>(st + 3 * X_TERM + off) = il;
      }
      fence_proxy_async();  // generic-proxy stores -> the MMA's async-proxy reads
      __syncwarp();
      if (lane == 0) arrive_remote(xfull0 + s * 8);
      ++cx;
      if (c == kcn - 1) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&sc_empty[sb]);
        ++it;
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        v[i][0] = vn[i][0];
        v[i][1] = vn[i][1];
      }
      t = tn;
      c = cn;
    }
  } else if (warp < WR_MMA) {
    // ------------------------------ epilogue ------------------------------
    // lane = bin 128 rank + 32 q + lane; columns = the tile's 128 signals
    const int q = warp - WR_EPI;
    const int bin = 128 * (int)rank + 32 * q + lane;
    const uint32_t acc_empty0 = mapa(smem_u32(acc_empty), 0);
    const uint32_t sc_empty_peer = mapa(smem_u32(sc_empty), peer);
    int it = 0;
    for (int64_t t = pair; t < ntiles; t += npairs, ++it) {
      const int ab = it & 1, sb = it % NSC;
      mbar_wait(&acc_full[ab], (it >> 1) & 1);
      wait_cluster(&sc_full[sb], (it / NSC) & 1);
      tmem_fence_after();
      const uint32_t base = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(ab * ACC_COLS);
      const float4* sc = scale + sb * TS;
#pragma unroll 1
      for (int s0 = 0; s0 < TS; s0 += 16) {
        uint32_t re[16], im[16];
        tmem_ld_re_im(base + (uint32_t)s0, base + (uint32_t)(TS + s0), re, im);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int64_t sig = t * TS + s0 + j;
          const float4 f = sc[s0 + j];  // broadcast read
          if (sig < p.batch && !(ASX_DTC2_ABLATE & 2))
            __stcs(reinterpret_cast<float2*>(p.X + sig * 2 * p.Xs) + bin,
                   make_float2(__uint_as_float(re[j]) * f.z * f.w, __uint_as_float(im[j]) * f.z * f.w));
        }
      }
      tmem_fence_before();
      __syncwarp();
      if (lane == 0) {
        arrive_remote(acc_empty0 + ab * 8);
        mbar_arrive(&sc_empty[sb]);
        arrive_cluster(sc_empty_peer + sb * 8);
      }
    }
  } else if (warp == WR_MMA) {
    // ------------------------------ MMA issuer (rank 0) ------------------------------
    if (rank == 0 && lane == 0) {
      uint32_t cx = 0, cw = 0;
      const uint32_t x0 = smem_u32(sX), w0 = smem_u32(sW);
      const uint32_t id = idesc2(false), idn = idesc2(true);
      int it = 0;
      for (int64_t t = pair; t < ntiles; t += npairs, ++it) {
        const int ab = it & 1;
        mbar_wait(&acc_empty[ab], ((it >> 1) & 1) ^ 1);
        tmem_fence_after();
        const uint32_t d_re = tmem + (uint32_t)(ab * ACC_COLS), d_im = d_re + (uint32_t)TS;
        for (int c = 0; c < kcn; ++c) {
          const uint32_t sw = cw % NW, sx = cx % NX;
          mbar_wait(&w_ready[sw], (cw / NW) & 1);
          mbar_wait(&x_full[sx], (cx / NX) & 1);
          tmem_fence_after();
          const uint32_t wrh = w0 + sw * W_STAGE, wrl = wrh + W_TERM, wih = wrl + W_TERM, wil = wih + W_TERM;
          const uint32_t xrh = x0 + sx * X_STAGE, xrl = xrh + X_TERM, xih = xrl + X_TERM, xil = xih + X_TERM;
#pragma unroll
          for (int k = 0; k < KC / 16 && !(ASX_DTC2_ABLATE & 1); ++k) {
            const uint32_t ko = k * 32;  // 16 fp16 along the 64-byte swizzled row
            const uint32_t first = (c == 0 && k == 0) ? 0u : 1u;
            // Re = Wr xr - Wi xi, Im = Wr xi + Wi xr, alternating between the two
            // accumulators so consecutive MMAs never wait on each other's D
            mma2_f16(d_re, dtc::sdesc(wrh + ko), dtc::sdesc(xrh + ko), id, first);
            mma2_f16(d_im, dtc::sdesc(wrh + ko), dtc::sdesc(xih + ko), id, first);
            mma2_f16(d_re, dtc::sdesc(wrh + ko), dtc::sdesc(xrl + ko), id, 1u);
            mma2_f16(d_im, dtc::sdesc(wrh + ko), dtc::sdesc(xil + ko), id, 1u);
            mma2_f16(d_re, dtc::sdesc(wrl + ko), dtc::sdesc(xrh + ko), id, 1u);
            mma2_f16(d_im, dtc::sdesc(wrl + ko), dtc::sdesc(xih + ko), id, 1u);
            mma2_f16(d_re, dtc::sdesc(wih + ko), dtc::sdesc(xih + ko), idn, 1u);
            mma2_f16(d_im, dtc::sdesc(wih + ko), dtc::sdesc(xrh + ko), id, 1u);
            mma2_f16(d_re, dtc::sdesc(wih + ko), dtc::sdesc(xil + ko), idn, 1u);
            mma2_f16(d_im, dtc::sdesc(wih + ko), dtc::sdesc(xrl + ko), id, 1u);
            mma2_f16(d_re, dtc::sdesc(wil + ko), dtc::sdesc(xih + ko), idn, 1u);
            mma2_f16(d_im, dtc::sdesc(wil + ko), dtc::sdesc(xrh + ko), id, 1u);
          }
          commit2(&w_empty[sw]);
          commit2(&x_empty[sx]);
          ++cw;
          ++cx;
        }
        commit2(&acc_full[ab]);
      }
    }
    __syncwarp();
  } else if (warp == WR_LOAD) {
    // ------------------------------ W loader ------------------------------
    if (lane == 0) {
      uint32_t cw = 0;
      for (int64_t t = pair; t < ntiles; t += npairs) {
        for (int c = 0; c < kcn; ++c, ++cw) {
          const uint32_t sw = cw % NW;
          mbar_wait(&w_empty[sw], ((cw / NW) & 1) ^ 1);
          if (ASX_DTC2_ABLATE & 16) {
            mbar_arrive(&w_full[sw]);
          } else {
            mbar_expect_tx(&w_full[sw], (uint32_t)W_STAGE);
            tma_load_1d(sW + sw * W_STAGE, p.wimg + (size_t)(2 * c + rank) * W_STAGE, (uint32_t)W_STAGE, &w_full[sw]);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == WR_RELAY) {
    // this CTA's W half has landed -> one arrival on rank 0's "W ready"
    if (lane == 0) {
      const uint32_t ready0 = mapa(smem_u32(w_ready), 0);
      uint32_t cw = 0;
      for (int64_t t = pair; t < ntiles; t += npairs) {
        for (int c = 0; c < kcn; ++c, ++cw) {
          const uint32_t sw = cw % NW;
          mbar_wait(&w_full[sw], (cw / NW) & 1);
          arrive_remote(ready0 + sw * 8);
        }
      }
    }
    __syncwarp();
  } else {
    // ------------------ per-signal scales, one tile ahead ------------------
    // 2^e, e = 10 - ilogb(max|x|), split e = e1 + e2 (asx_direct_tc.cuh); the
    // CTA's 64 signals, 8 per warp, four at a time with all loads in flight
    // (this first read of x comes from HBM: eight warps keep enough of it in flight)
    const int sw = warp - WR_SCALE;
    const uint32_t sc_full_peer = mapa(smem_u32(sc_full), peer);
    int it = 0;
    for (int64_t t = pair; t < ntiles; t += npairs, ++it) {
      const int sb = it % NSC;
      wait_cluster(&sc_empty[sb], ((it / NSC) & 1) ^ 1);
      float4* sc = scale + sb * TS;
      const uint32_t sc_peer = mapa(smem_u32(sc), peer);
      for (int r0 = 8 * sw; r0 < 8 * sw + 8; r0 += 4) {
        float mx[4] = {0.f, 0.f, 0.f, 0.f};
        const int nq = p.n / 2;  // float4 per row
        for (int i0 = 0; i0 < nq; i0 += 128) {
          float4 v[4][4];
#pragma unroll
          for (int rr = 0; rr < 4; ++rr) {
            const int64_t b = t * TS + HS * rank + r0 + rr;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int i = i0 + lane + 32 * u;
              v[rr][u] = make_float4(0.f, 0.f, 0.f, 0.f);
              if (b < p.batch && i < nq && !(ASX_DTC2_ABLATE & 8)) v[rr][u] = __ldg(reinterpret_cast<const float4*>(p.x + b * 2 * p.xs) + i);
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
            int e = 0;
            if (mx[rr] > 0.f && mx[rr] <= 3.402823466e38f) e = 10 - ilogbf(mx[rr]);
            const int e1 = e / 2;
            const float f1 = exp2f((float)e1), f2 = exp2f((float)(e - e1));
            const float4 val = make_float4(f1, f2, 1.f / f1, 1.f / (f2 * W_SCALE));
            const int slot = HS * (int)rank + r0 + rr;
            sc[slot] = val;
            st_cluster_f4(sc_peer + slot * 16, val);
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
        asm volatile("fence.acq_rel.cluster;" ::: "memory");  // the warp's local + remote scale stores
        arrive_cluster(mapa(smem_u32(&sc_full[sb]), rank));
        arrive_cluster(sc_full_peer + sb * 8);
      }
    }
  }
  tmem_fence_before();
  cluster_sync();  // no CTA leaves (or deallocates) while its peer may still touch it
  tmem_fence_after();
  if (warp == WR_MMA) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

// Plan time: the pair layout of the W image, [chunk][cta r][Wr hi | Wr lo |
// Wi hi | Wi lo][128 bins][32] fp16 in K-major SWIZZLE_64B, CTA r's half =
// bins 128r..128r+127 (one 32 KB bulk copy per chunk per CTA).
__global__ void k_direct_tc2_image(unsigned char* img, int n, uint64_t a, uint64_t L) {
  const int64_t total = (int64_t)n * MB;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int mb = (int)(e / n), nn = (int)(e % n);
    const uint64_t ph = (uint64_t)(((unsigned __int128)((uint64_t)a * (uint64_t)mb) * (uint64_t)nn) % L);
    double sn, cs;
    sincospi(2.0 * (double)ph / (double)L, &sn, &cs);  // W = cs - i sn
    const double w[2] = {cs * (double)W_SCALE, -sn * (double)W_SCALE};
    const int c = nn / KC, k = nn % KC, r = mb >> 7, row = mb & 127;
    const uint32_t off = dtc::swz((uint32_t)row, (uint32_t)k);
    unsigned char* st = img + (size_t)(2 * c + r) * W_STAGE;
#pragma unroll
    for (int part = 0; part < 2; ++part) {
      const __half hi = __float2half_rn((float)w[part]);
      const __half lo = __float2half_rn((float)(w[part] - (double)__half2float(hi)));
      *reinterpret_cast<__half*>(st + (2 * part) * W_TERM + off) = hi;
      *reinterpret_cast<__half*>(st + (2 * part + 1) * W_TERM + off) = lo;
    }
  }
}

}  // namespace dtc2
}  // namespace asx

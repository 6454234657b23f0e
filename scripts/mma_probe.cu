// mma_probe.cu — tcgen05.mma kind::f16 issue-rate probe (SS operands, K-major
// SWIZZLE_64B, the layout k_direct_tc uses) for cta_group::1 vs ::2 and N.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_probe scripts/mma_probe.cu
// Run:   ./mma_probe  -> cycles per MMA instruction, per-SM MAC rate, for each shape,
//        alone and with 8 warps streaming shared-memory stores beside the MMAs.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}
__device__ __forceinline__ uint32_t idesc(int m, int n) {
  return (1u << 4) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

template <int CG, int M, int N, int NOISE>
__global__ void __launch_bounds__(320, 1) probe(int groups, unsigned long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* s = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  // [A 8 KB x 4 | B 16 KB x 4 | noise 32 KB | bars]
  unsigned char* sA = s;
  unsigned char* sB = s + 4 * 8192;
  float* noise = reinterpret_cast<float*>(s + 4 * 8192 + 4 * 16384);
  uint64_t* bar = reinterpret_cast<uint64_t*>(s + 4 * 8192 + 4 * 16384 + 32768);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (4 * 8192 + 4 * 16384) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (CG == 2) {
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;");
  } else {
    __syncthreads();
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *slot;
  const bool leader = CG == 1 || cta_rank() == 0;
  if (warp == 8 && (threadIdx.x & 31) == 0 && leader) {
    const uint32_t id = idesc(M, N);
    const uint32_t a0 = su32(sA), b0 = su32(sB);
    unsigned long long t0 = clock64();
    uint32_t ph = 0;
    for (int g = 0; g < groups; ++g) {
      for (int j = 0; j < 24; ++j) {
        const uint32_t st = j & 3;
        const uint64_t da = sdesc(a0 + st * 8192 + (j & 1) * 32), db = sdesc(b0 + st * 16384 + (j & 1) * 32);
        const uint32_t d = tmem + ((j & 1) ? (uint32_t)N : 0u);
        if (CG == 1)
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
                       "l"(da), "l"(db), "r"(id), "r"(1));
        else
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
                       "l"(da), "l"(db), "r"(id), "r"(1));
      }
      if (CG == 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)));
      else
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(su32(bar)),
                     "h"((uint16_t)3));
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(su32(bar)), "r"(ph));
      ph ^= 1;
    }
    cyc[blockIdx.x] = clock64() - t0;
  } else if (NOISE && warp < 8) {
    // converter-like traffic: 16-byte stores streaming over 32 KB, ~the k_direct_tc converter rate
    float4* nz = reinterpret_cast<float4*>(noise);
    const float4 v = make_float4(1.f, 2.f, 3.f, 4.f);
    for (int g = 0; g < groups; ++g)
      for (int i = threadIdx.x; i < 2048; i += 256) nz[i] = v;
  } else if (CG == 2 && !leader && warp == 8 && (threadIdx.x & 31) == 0) {
    // follower: wait for the leader's multicast commits so teardown is ordered
    uint32_t ph = 0;
    for (int g = 0; g < groups; ++g) {
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(su32(bar)), "r"(ph));
      ph ^= 1;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (CG == 2) {
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;");
  } else {
    __syncthreads();
  }
  if (warp == 0) {
    if (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int CG, int M, int N, int NOISE>
void run(const char* name) {
  const int groups = 2000, sms = 148;
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long) * sms);
  cudaMemset(d, 0, sizeof(unsigned long long) * sms);
  const int smem = 1024 + 4 * 8192 + 4 * 16384 + 32768 + 64;
  auto k = probe<CG, M, N, NOISE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(320);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, k, groups, d);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k, groups, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  const double mmas = 24.0 * groups;
  const double macs_per_sm = mmas * M * N * 16.0 / CG;
  printf("%-34s err=%s  %.1f cyc/MMA  %.0f MAC/cyc/SM  %.1f TFLOP/s (fp16 dense, events %.3f ms)\n", name,
         cudaGetErrorString(err), mx / mmas, macs_per_sm / (mx / 1.0) * 1.0,
         2.0 * macs_per_sm * sms / (ms / 1e3) / 1e12, ms);
  cudaFree(d);
}

int main() {
  run<1, 128, 256, 0>("cta_group::1 M128 N256");
  run<1, 128, 128, 0>("cta_group::1 M128 N128");
  run<1, 128, 64, 0>("cta_group::1 M128 N64");
  run<1, 128, 32, 0>("cta_group::1 M128 N32");   // a radix-16 complex DFT pass as a real GEMM: N = 32
  run<1, 128, 16, 0>("cta_group::1 M128 N16");
  run<1, 64, 256, 0>("cta_group::1 M64 N256");
  run<1, 64, 128, 0>("cta_group::1 M64 N128");
  run<1, 64, 32, 0>("cta_group::1 M64 N32");
  run<2, 256, 256, 0>("cta_group::2 M256 N256");
  run<2, 256, 128, 0>("cta_group::2 M256 N128");
  run<1, 128, 256, 1>("cta_group::1 M128 N256 + smem stores");
  run<2, 256, 256, 1>("cta_group::2 M256 N256 + smem stores");
  run<2, 256, 128, 1>("cta_group::2 M256 N128 + smem stores");
  return 0;
}

// Per-SM global-store throughput probe (B200): how fast can ONE SM push data to
// L2 / HBM with st.global.v4 from registers vs cp.async.bulk shared -> global?
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o store_bw scripts/store_bw.cu && ./store_bw
// Prints bytes per SM clock per SM for: all SMs / a quarter of the SMs writing,
// footprint inside L2 (each CTA rewrites 256 KiB) / streaming to HBM (4 MiB per CTA).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>  // 0: st.global.cs.v4, 1: cp.async.bulk shared -> global (32 KiB pieces)
__global__ void __launch_bounds__(256, 1) k_store(float4* out, size_t region_f4, int pieces, int reps, long long* cyc) {
  extern __shared__ __align__(128) unsigned char sm[];
  float4* dst = out + (size_t)blockIdx.x * region_f4;
  const int tid = threadIdx.x;
  if (MODE == 1) {
    for (int i = tid; i < 2048; i += 256) reinterpret_cast<float4*>(sm)[i] = make_float4(i, 1.f, 2.f, 3.f);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    for (int pc = 0; pc < pieces; ++pc) {  // one piece = 32 KiB = 2048 float4
      float4* d = dst + (size_t)pc * 2048;
      if (MODE == 0) {
#pragma unroll
        for (int k = 0; k < 8; ++k) __stcs(d + tid + 256 * k, make_float4(r, pc, k, tid));
      } else if (tid == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 32768;" ::"l"(d), "r"(smem_u32(sm)) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
      }
    }
  }
  if (MODE == 1 && tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  __syncthreads();
  if (tid == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t big = (size_t)sms * (4u << 20);
  float4* out;
  long long* cyc;
  cudaMalloc(&out, big);
  cudaMalloc(&cyc, sms * sizeof(long long));
  cudaFuncSetAttribute(k_store<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  long long* h = new long long[sms];
  for (int mode = 0; mode < 2; ++mode)
    for (int frac = 1; frac <= 4; frac *= 4)
      for (int hbm = 0; hbm < 2; ++hbm) {
        const int grid = sms / frac;
        const int pieces = hbm ? 128 : 8;   // 4 MiB or 256 KiB per CTA
        const int reps = hbm ? 4 : 64;
        const size_t region_f4 = (size_t)(4u << 20) / 16;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int it = 0; it < 2; ++it) {
          cudaEventRecord(e0);
          if (mode == 0)
            k_store<0><<<grid, 256, 0>>>(out, region_f4, pieces, reps, cyc);
          else
            k_store<1><<<grid, 256, 32768>>>(out, region_f4, pieces, reps, cyc);
          cudaEventRecord(e1);
          cudaDeviceSynchronize();
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaMemcpy(h, cyc, grid * sizeof(long long), cudaMemcpyDeviceToHost);
        double mean = 0;
        for (int i = 0; i < grid; ++i) mean += (double)h[i];
        mean /= grid;
        const double bytes = (double)pieces * 32768.0 * reps;
        printf("%-28s %3d CTAs, %s: %.1f B/clk/SM, aggregate %.2f TB/s (err=%s)\n",
               mode ? "cp.async.bulk smem->global" : "st.global.cs.v4 (registers)", grid,
               hbm ? "4 MiB/CTA streaming (HBM)" : "256 KiB/CTA rewritten (L2) ", bytes / mean,
               bytes * grid / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}

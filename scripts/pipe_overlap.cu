// Do FP64 arithmetic and shared-memory accesses overlap on one SM?  (B200 probe)
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o pipe_overlap scripts/pipe_overlap.cu
// One 512-thread CTA per SM.  "math" warps run a chain-free stream of DFMA (or
// FFMA), "lds" warps a stream of conflict-free 16-byte shared-memory loads.
// Rows: all 16 warps math / all 16 warps lds / 8 warps each.  If the two
// streams use independent pipes the mixed run takes max(math/2, lds/2); if
// they share an issue path it takes math/2 + lds/2.
#include <cstdio>
#include <cuda_runtime.h>

template <typename T>
__device__ __forceinline__ void math_stream(int iters, T* out) {
  T a0 = 1, a1 = 2, a2 = 3, a3 = 4, a4 = 5, a5 = 6, a6 = 7, a7 = 8;
  const T m = T(1.0000001), c = T(1e-9);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      a0 = a0 * m + c; a1 = a1 * m + c; a2 = a2 * m + c; a3 = a3 * m + c;
      a4 = a4 * m + c; a5 = a5 * m + c; a6 = a6 * m + c; a7 = a7 * m + c;
    }
  }
  out[threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__device__ __forceinline__ void lds_stream(int iters, const double2* sm, double* out) {
  unsigned x0 = 0, x1 = 0, x2 = 0, x3 = 0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const double2* p = sm + w * 256 + lane;  // 8 x 512 contiguous bytes per warp
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      unsigned a, b, c, d;
      asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                   : "r"((unsigned)__cvta_generic_to_shared(p + 32 * k)), "r"(i));
      x0 ^= a; x1 ^= b; x2 ^= c; x3 ^= d;  // integer XORs keep the loads live without touching the FP pipes
    }
  }
  out[threadIdx.x] = (double)(x0 ^ x1 ^ x2 ^ x3);
}

// mode: 0 all math, 1 all lds, 2 warps 0-7 math + 8-15 lds
template <typename T>
__global__ void __launch_bounds__(512, 1) k(int mode, int it_math, int it_lds, T* outm, double* outl, long long* cyc) {
  extern __shared__ double2 sm[];  // 16 warps x 256 elements = 64 KiB
  for (int i = threadIdx.x; i < 16 * 256; i += 512) sm[i] = make_double2(i, 1.0);
  __syncthreads();
  const long long t0 = clock64();
  const int w = threadIdx.x >> 5;
  const bool math = mode == 0 || (mode == 2 && w < 8);
  if (math) math_stream<T>(it_math, outm + blockIdx.x * 512);
  else lds_stream(it_lds, sm, outl + blockIdx.x * 512);
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

template <typename T>
void run(const char* name, int it_math, int it_lds) {
  T* om; double* ol; long long* cyc;
  cudaMalloc(&om, 148 * 512 * sizeof(T)); cudaMalloc(&ol, 148 * 512 * sizeof(double)); cudaMalloc(&cyc, 148 * 8);
  long long h[148];
  double res[3];
  for (int mode = 0; mode < 3; ++mode) {
    cudaFuncSetAttribute(k<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    for (int r = 0; r < 2; ++r) k<T><<<148, 512, 65536>>>(mode, it_math, it_lds, om, ol, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double s = 0; for (int i = 0; i < 148; ++i) s += h[i];
    res[mode] = s / 148;
  }
  printf("%s: all-math %.0f cyc, all-lds %.0f cyc, 8 warps each %.0f cyc  (independent pipes: %.0f, shared path: %.0f)  err=%s\n",
         name, res[0], res[1], res[2], res[0] / 2 > res[1] / 2 ? res[0] / 2 : res[1] / 2, res[0] / 2 + res[1] / 2,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  // iteration counts chosen so both streams alone take about the same time
  run<double>("DFMA vs ld.shared 16 B/lane", 400, 400);
  run<float>("FFMA vs ld.shared 16 B/lane", 800, 400);
  return 0;
}

// fp_peaks.cu — measured FP32 (FFMA) and FP64 (DFMA) peak throughput of this
// GPU, the compute-side roofline denominators for the FP-bound configs
// (SURVEY.md §8d asks for them; MEASURED_PEAKS.json has only HBM and bf16).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/fp_peaks scripts/fp_peaks.cu
//   build/fp_peaks > profiles/fp_peaks.json
//
// Each thread runs CH independent FMA chains (enough ILP to cover the FMA
// latency), grid = SMs x 8 CTAs of 256 threads, best of 10 timed launches.
#include <cstdio>
#include <cuda_runtime.h>

template <typename T, int CH>
__global__ void __launch_bounds__(256) k_fma(T* out, int iters, T a, T b) {
  T v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = T(threadIdx.x + c) * T(1e-3);
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int c = 0; c < CH; ++c) v[c] = fma(v[c], a, b);
    }
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += v[c];
  if (s == T(12345.678)) out[0] = s;  // keeps the chains live
}

// packed FP32x2 (FFMA2): same lane count, half the issue slots
template <int CH>
__global__ void __launch_bounds__(256) k_fma2(float* out, int iters, float a, float b) {
  float2 v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = make_float2(float(threadIdx.x + c) * 1e-3f, float(c) * 1e-3f);
  const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int c = 0; c < CH; ++c) v[c] = __ffma2_rn(v[c], a2, b2);
    }
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += v[c].x + v[c].y;
  if (s == 12345.678f) out[0] = s;
}

template <typename T, int CH, bool PACKED = false>
double run(int sms, int iters) {
  T* out;
  cudaMalloc(&out, sizeof(T));
  const int grid = sms * 8, block = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto launch = [&]() {
    if constexpr (PACKED)
      k_fma2<CH><<<grid, block>>>(reinterpret_cast<float*>(out), iters, 0.999999f, 1e-7f);
    else
      k_fma<T, CH><<<grid, block>>>(out, iters, T(0.999999), T(1e-7));
  };
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaFree(out);
  const double flops = 2.0 * double(grid) * block * iters * 16 * CH * (PACKED ? 2 : 1);
  return flops / (best * 1e-3) / 1e12;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const double f32 = run<float, 8>(sms, 4096);
  const double f64 = run<double, 8>(sms, 1024);
  const double f32x2 = run<float, 8, true>(sms, 4096);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
    return 1;
  }
  printf("{\"fp32_tflops\": %.2f, \"fp32x2_tflops\": %.2f, \"fp64_tflops\": %.2f, \"sms\": %d, \"max_clock_mhz\": %.0f, "
         "\"fp32_nominal_tflops\": %.2f, \"fp64_nominal_tflops\": %.2f, "
         "\"how\": \"FFMA/DFMA, FFMA2 (packed), 8 independent chains per thread, grid SMs x 8 x 256, best of 10 CUDA-event timings\"}\n",
         f32, f32x2, f64, sms, clk / 1e3, sms * 128 * 2.0 * clk * 1e3 / 1e12, sms * 64 * 2.0 * clk * 1e3 / 1e12);
  return 0;
}

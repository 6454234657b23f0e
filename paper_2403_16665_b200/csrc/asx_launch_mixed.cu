// asx_launch_mixed.cu — the complex64 α-FFT: FP64 recursion (the kernels of
// asx_launch_f64.cu's α-FFT family) with complex64 / float32 signal rows and
// complex64 bins, so the paper's recursion meets the complex64 bound on every
// input the complex128 path does.
#include "asx_dispatch.cuh"

namespace asx_host {

cudaError_t launch_afft_io32(int P, const KParams& kp, int64_t batch, cudaStream_t st, const LaunchEnv& env) {
  switch (P) {
#define ASX_MIXED(S) \
  case S:            \
    return launch_persist<double, S, KIND_AFFT, float>(kp, batch, st, env);
    ASX_MIXED(1)
    ASX_MIXED(2)
    ASX_MIXED(4)
    ASX_MIXED(8)
    ASX_MIXED(16)
    ASX_MIXED(32)
    ASX_MIXED(64)
    ASX_MIXED(128)
    ASX_MIXED(256)
    ASX_MIXED(512)
    ASX_MIXED(1024)
    ASX_MIXED(2048)
    ASX_MIXED(4096)
    ASX_MIXED(8192)
#undef ASX_MIXED
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace asx_host

// asx_launch_misc.cu — non-template launch helpers (four-step path, the
// opt-in two-halves chirp kernel) and the per-thread last-launch record.
#include "asx_dispatch.cuh"

namespace asx_host {

thread_local LastLaunch g_last_launch;

cudaError_t launch_large(int dbl, int64_t P1, int mode_cols, int mode_rows, int which, const LParams& lp,
                         cudaStream_t st) {
  // which: 0 = cols, 1 = rows
  if (which == 0) return dbl ? launch_cols_p1<double>(P1, mode_cols, lp, st) : launch_cols_p1<float>(P1, mode_cols, lp, st);
  return dbl ? launch_rows<double>(mode_rows, P1, lp, st) : launch_rows<float>(mode_rows, P1, lp, st);
}

// Resident CTAs per SM of the two-halves kernel for this precision (0 if n/a).
int chirp2h_occupancy(int dbl) {
  int v = 0;
  if (dbl) {
    auto k = chirp2h_kernel<double, 4096, 512>();
    using G = Chirp2hCfg<double, 4096, 512>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k, 512, G::SMEM) != cudaSuccess)
      v = 0;
  } else {
    auto k = chirp2h_kernel<float, 8192, 512>();
    using G = Chirp2hCfg<float, 8192, 512>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k, 512, G::SMEM) != cudaSuccess)
      v = 0;
  }
  cudaGetLastError();
  if (const char* f = std::getenv("ASX_2H_PER_SM")) v = std::atoi(f);  // tuning override
  return v;
}

cudaError_t launch_chirp2h(int dbl, const KParams& kp, int grid, void* scratch, const void* cw, const void* cwc,
                           cudaStream_t st) {
  if (dbl) {
    using G = Chirp2hCfg<double, 4096, 512>;
    k_chirp2h<double, 4096, 512><<<grid, 512, G::SMEM, st>>>(kp, scratch, cw, cwc);
  } else {
    using G = Chirp2hCfg<float, 8192, 512>;
    k_chirp2h<float, 8192, 512><<<grid, 512, G::SMEM, st>>>(kp, scratch, cw, cwc);
  }
  g_last_launch.grid = grid;
  g_last_launch.block = 512;
  g_last_launch.smem = (int)(dbl ? Chirp2hCfg<double, 4096, 512>::SMEM : Chirp2hCfg<float, 8192, 512>::SMEM);
  g_last_launch.staged = 4;  // bit 2: two-halves kernel
  g_last_launch.tmem = 1;
  return cudaGetLastError();
}

}  // namespace asx_host

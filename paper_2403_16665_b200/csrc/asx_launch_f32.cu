// asx_launch_f32.cu — instantiates every float kernel of the FFT family
// (persistent α-FFT / chirp-z, four-step columns and rows).
#include "asx_dispatch.cuh"

namespace asx_host {
template cudaError_t launch_by_size<float>(int, int, const KParams&, int64_t, cudaStream_t, const LaunchEnv&);
template cudaError_t launch_cols_p1<float>(int64_t, int, const LParams&, cudaStream_t);
template cudaError_t launch_rows<float>(int, int64_t, const LParams&, cudaStream_t);
}  // namespace asx_host

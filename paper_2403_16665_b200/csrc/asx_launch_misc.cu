// asx_launch_misc.cu — non-template launch helpers (four-step path) and the
// per-thread last-launch record.
#include "asx_dispatch.cuh"

namespace asx_host {

thread_local LastLaunch g_last_launch;

cudaError_t launch_large(int dbl, int64_t P1, int mode_cols, int mode_rows, int which, const LParams& lp,
                         cudaStream_t st) {
  // which: 0 = cols, 1 = rows
  if (which == 0) return dbl ? launch_cols_p1<double>(P1, mode_cols, lp, st) : launch_cols_p1<float>(P1, mode_cols, lp, st);
  return dbl ? launch_rows<double>(mode_rows, P1, lp, st) : launch_rows<float>(mode_rows, P1, lp, st);
}

}  // namespace asx_host

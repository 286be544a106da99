// rsw_pipe_256.cu — the pipelined parareal kernels (rsw_pipeline.cuh) instantiated for n = 256
// (one translation unit per n, compiled in parallel).
#include "rsw_pipeline.cuh"

namespace rsw {
cudaError_t launch_parareal_pipe_256(const PipeArgs& a, int fine_scheme, int grid, size_t* out, cudaStream_t st) {
  return launch_pipe_n<256>(a, fine_scheme, grid, out, st);
}
}  // namespace rsw

// rsw_pipeline.cu — dispatch of the pipelined parareal megakernel (rsw_pipeline.cuh)
// to its per-n translation units rsw_pipe_{64,128,256}.cu.
#include "rsw_internal.h"

namespace rsw {

cudaError_t launch_parareal_pipe_64(const PipeArgs& a, int fine_scheme, int grid, size_t* out, cudaStream_t st);
cudaError_t launch_parareal_pipe_128(const PipeArgs& a, int fine_scheme, int grid, size_t* out, cudaStream_t st);
cudaError_t launch_parareal_pipe_256(const PipeArgs& a, int fine_scheme, int grid, size_t* out, cudaStream_t st);

bool pipeline_supported(int n) { return n == 64 || n == 128 || n == 256; }

// grid <= 0: return the number of co-resident CTAs in *out (capacity query)
cudaError_t launch_parareal_pipe(int n, const PipeArgs& a, int fine_scheme, int grid, size_t* out,
                                 cudaStream_t st) {
  switch (n) {
    case 64: return launch_parareal_pipe_64(a, fine_scheme, grid, out, st);
    case 128: return launch_parareal_pipe_128(a, fine_scheme, grid, out, st);
    case 256: return launch_parareal_pipe_256(a, fine_scheme, grid, out, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace rsw

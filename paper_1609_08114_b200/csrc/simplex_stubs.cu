// Temporary stubs for size classes not compiled yet.
#include "lpb_internal.cuh"
namespace lpb {
bool thread_fits(int, int) { return false; }
cudaError_t launch_simplex_thread(const SimplexArgs&, int, cudaStream_t) { return cudaErrorNotSupported; }
bool reg_fits(int, int, int) { return false; }
cudaError_t launch_simplex_reg(const SimplexArgs&, int, cudaStream_t, int*) { return cudaErrorNotSupported; }
}

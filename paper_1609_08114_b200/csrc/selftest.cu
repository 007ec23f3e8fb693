// selftest.cu — diagnostic kernels behind include/lpb_selftest.h.
#include "../../include/lpb.h"
#include "../../include/lpb_selftest.h"
#include "lpb_fp64.cuh"

namespace {
__global__ void div_check(const double* a, const double* b, double* q, int64_t n,
                          unsigned long long* cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    bool slow;
    double f = lpb::div_fast(a[i], b[i], slow);
    if (slow) f = __ddiv_rn(a[i], b[i]);
    const double r = __ddiv_rn(a[i], b[i]);
    q[i] = f;
    if (__double_as_longlong(f) != __double_as_longlong(r)) atomicAdd(cnt, 1ull);
    if (slow) atomicAdd(cnt + 1, 1ull);
  }
}
}  // namespace

extern "C" int lpb_selftest_div(const double* a, const double* b, double* q, int64_t n,
                                int64_t* out) {
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, 2 * sizeof(unsigned long long)) != cudaSuccess) return LPB_ECUDA;
  cudaMemset(d, 0, 2 * sizeof(unsigned long long));
  div_check<<<1024, 256>>>(a, b, q, n, d);
  unsigned long long h[2] = {0, 0};
  const cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return LPB_ECUDA;
  out[0] = (int64_t)h[0];
  out[1] = (int64_t)h[1];
  return LPB_OK;
}

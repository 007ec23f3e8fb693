// DFMA throughput vs resident warps per SM (one CTA per SM), ILP 8 or 16 independent chains.
#include <cstdio>
template <int ILP>
__global__ void k(double* out, int iters) {
  double a[ILP];
#pragma unroll
  for (int u = 0; u < ILP; ++u) a[u] = threadIdx.x * 1e-3 + u;
  const double m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int u = 0; u < ILP; ++u) a[u] = __fma_rn(a[u], m, c);
  }
  double s = 0;
#pragma unroll
  for (int u = 0; u < ILP; ++u) s += a[u];
  if (s == 12345.0) out[0] = s;
}
template <int ILP>
void run(int sms, int wps, double* d) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2048;
  k<ILP><<<sms, 32 * wps>>>(d, 16);
  cudaEventRecord(e0);
  k<ILP><<<sms, 32 * wps>>>(d, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 2.0 * 4 * ILP * (double)iters * sms * 32 * wps;
  const double instr_per_clk_sm = (4.0 * ILP * iters * wps) / (ms * 1e-3 * 1.965e9);
  printf("ILP %2d warps/SM %2d: %7.2f TFLOP/s  warp-DFMA/clk/SM %.3f  per-warp issue interval %.2f clk\n",
         ILP, wps, fl / (ms * 1e-3) / 1e12, instr_per_clk_sm, wps / instr_per_clk_sm);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d; cudaMalloc(&d, 64);
  for (int w : {1, 2, 4, 8, 16, 32}) { run<8>(sms, w, d); run<16>(sms, w, d); }
  return 0;
}

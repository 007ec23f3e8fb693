// Throughput of the fp64 reciprocal seed on sm_100: MUFU.RCP64H (rcp.approx.ftz.f64) vs an
// fp32 seed (F2F + MUFU.RCP + F2F), many warps, 8 independent chains per thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_tp mufu_tp.cu && ./mufu_tp
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k64(double* out, int iters) {
  double v[8];
  for (int i = 0; i < 8; ++i) v[i] = 1.0 + threadIdx.x * 1e-3 + i;
  for (int t = 0; t < iters; ++t)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double r;
      asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(v[i]));
      v[i] = r + 1.0;
    }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k32(double* out, int iters) {
  double v[8];
  for (int i = 0; i < 8; ++i) v[i] = 1.0 + threadIdx.x * 1e-3 + i;
  for (int t = 0; t < iters; ++t)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float f = __double2float_rn(v[i]);
      float r;
      asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f));
      v[i] = (double)r + 1.0;
    }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void kdfma(double* out, int iters) {
  double v[8];
  for (int i = 0; i < 8; ++i) v[i] = 1.0 + threadIdx.x * 1e-3 + i;
  for (int t = 0; t < iters; ++t)
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __fma_rn(v[i], 0.999, 1.0);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 16 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 2000;
  for (int warps : {4, 8, 16, 32}) {
    const int nt = 32 * warps;
    for (int which = 0; which < 3; ++which) {
      auto launch = [&]() {
        if (which == 0) k64<<<sms, nt>>>(out, iters);
        else if (which == 1) k32<<<sms, nt>>>(out, iters);
        else kdfma<<<sms, nt>>>(out, iters);
      };
      launch();
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double ops = (double)sms * nt * iters * 8;
      printf("warps/SM %2d  %-10s %8.2f Gop/s  %6.2f lane-ops/clk/SM (1.965 GHz)\n", warps,
             which == 0 ? "rcp64h" : which == 1 ? "f32-seed" : "dfma", ops / ms / 1e6,
             ops / (ms * 1e-3) / 1.965e9 / sms);
    }
  }
  return 0;
}

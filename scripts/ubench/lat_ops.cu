// Dependent-chain latency of the operations on the simplex kernels' critical path (cycles per
// step, one warp alone on an SM; 128 threads for the barrier).  nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 lat_ops.cu -o lat_ops && ./lat_ops
#include <cstdio>
constexpr int IT = 4096;
__global__ void k(double* io, long long* out) {
  const int lane = threadIdx.x & 31;
  double d = io[threadIdx.x];
  unsigned u = (unsigned)threadIdx.x * 2654435761u;
  long long t0, t1;
  __shared__ double sm[256];
  // REDUX (__reduce_max_sync) chain
  t0 = clock64();
  for (int i = 0; i < IT; ++i) u = __reduce_max_sync(0xffffffffu, u + (unsigned)i) ^ (unsigned)lane;
  t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / IT;
  // SHFL (index) chain on a double
  t0 = clock64();
  for (int i = 0; i < IT; ++i) d = __shfl_sync(0xffffffffu, d, (lane + 1) & 31) + 1.0;
  t1 = clock64();
  if (threadIdx.x == 0) out[1] = (t1 - t0) / IT;
  // MUFU.RCP64H chain
  t0 = clock64();
  for (int i = 0; i < IT; ++i) {
    double r;
    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    d = r + 1.0;
  }
  t1 = clock64();
  if (threadIdx.x == 0) out[2] = (t1 - t0) / IT;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < IT; ++i) d = __fma_rn(d, 0.999, 1e-3);
  t1 = clock64();
  if (threadIdx.x == 0) out[3] = (t1 - t0) / IT;
  // BALLOT + FFS chain
  t0 = clock64();
  for (int i = 0; i < IT; ++i) u = __ffs(__ballot_sync(0xffffffffu, ((u + lane) & 3) == 0)) + u;
  t1 = clock64();
  if (threadIdx.x == 0) out[4] = (t1 - t0) / IT;
  // STS -> LDS round trip (same thread)
  t0 = clock64();
  for (int i = 0; i < IT; ++i) {
    sm[threadIdx.x] = d;
    __syncwarp();
    d = sm[(threadIdx.x + 1) & 31] + 1.0;
  }
  t1 = clock64();
  if (threadIdx.x == 0) out[5] = (t1 - t0) / IT;
  // __syncthreads (128 threads) with a dependent SMEM exchange
  t0 = clock64();
  for (int i = 0; i < IT; ++i) {
    sm[threadIdx.x] = d;
    __syncthreads();
    d = sm[(threadIdx.x + 32) & 127] + 1.0;
    __syncthreads();
  }
  t1 = clock64();
  if (threadIdx.x == 0) out[6] = (t1 - t0) / (2 * IT);
  // division fast path (rcp + 2 Newton + residual) chain
  t0 = clock64();
  for (int i = 0; i < IT; ++i) d = __ddiv_rn(1.0 + d, 3.0 + (double)i);
  t1 = clock64();
  if (threadIdx.x == 0) out[7] = (t1 - t0) / IT;
  io[threadIdx.x] = d + (double)u;
}
int main() {
  double* io;
  long long* out;
  cudaMalloc(&io, 256 * 8);
  cudaMemset(io, 0, 256 * 8);
  cudaMalloc(&out, 16 * 8);
  k<<<1, 128>>>(io, out);
  k<<<1, 128>>>(io, out);
  long long h[16];
  cudaMemcpy(h, out, 16 * 8, cudaMemcpyDeviceToHost);
  const char* nm[] = {"REDUX.max (+iadd)", "SHFL.idx f64 (+dadd)", "MUFU.RCP64H (+dadd)",
                      "DFMA", "VOTE.ballot+FLO (+iadd)", "STS->LDS (+syncwarp, dadd)",
                      "BAR.SYNC 128 thr (+LDS/STS)", "__ddiv_rn (+dadd)"};
  for (int i = 0; i < 8; ++i) printf("%-30s %lld cycles/step\n", nm[i], h[i]);
  return 0;
}

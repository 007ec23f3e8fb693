// tmem_bw.cu — TMEM load/store throughput from ordinary warps (tcgen05.ld/st 32x32b.x16),
// the question being whether TMEM can hold part of a register-class tableau.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw tmem_bw.cu && ./tmem_bw
// Each CTA (4 warps = 128 TMEM lanes) allocates NCOL columns and repeatedly loads, updates
// (one DFMA per 64-bit pair) and stores them; CTAs per SM = 1..4.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int NCOL>
__global__ void __launch_bounds__(128) tm_kernel(int iters, long long* cyc, double* sink, int rw) {
  __shared__ uint32_t taddr_s;
  const int w = threadIdx.x >> 5;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&taddr_s)), "n"(NCOL));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t base = taddr_s + ((uint32_t)(w * 32) << 16);
  uint32_t v[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = 0u;
#pragma unroll 1
  for (int c = 0; c < NCOL; c += 16)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
                 ::"r"(base + c), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                 "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
  asm volatile("tcgen05.wait::st.sync.aligned;\n");
  __syncthreads();
  const long long t0 = clock64();
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 1
    for (int c = 0; c < NCOL; c += 16) {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                     "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                   : "r"(base + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
      for (int k = 0; k < 16; k += 2) {
        double d = __hiloint2double((int)v[k + 1], (int)v[k]);
        d = __fma_rn(d, 1.0000001, 1e-300);
        acc += d;
        v[k] = (uint32_t)__double2loint(d);
        v[k + 1] = (uint32_t)__double2hiint(d);
      }
      if (rw)
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
                     ::"r"(base + c), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                     "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * 128 + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr_s), "n"(NCOL));
}

template <int NCOL>
void run(int per_sm, int rw) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * per_sm, iters = 200;
  long long* cyc;
  double* sink;
  cudaMalloc(&cyc, grid * sizeof(long long));
  cudaMalloc(&sink, grid * 128 * sizeof(double));
  tm_kernel<NCOL><<<grid, 128>>>(iters, cyc, sink, rw);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  tm_kernel<NCOL><<<grid, 128>>>(iters, cyc, sink, rw);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h = 0;
  cudaMemcpy(&h, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
  const double bytes_per_cta = (double)iters * NCOL * 128 * 4;  // read (and write if rw)
  const double per_sm_bytes = bytes_per_cta * per_sm;
  printf("NCOL %3d CTAs/SM %d %s: %s  cta cycles %lld -> %.1f B/cycle/SM read (%.2f TB/s chip read)\n",
         NCOL, per_sm, rw ? "ld+st" : "ld   ", cudaGetErrorString(err), h,
         per_sm_bytes / (double)h, bytes_per_cta * grid / (ms * 1e-3) / 1e12);
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  for (int rw = 0; rw < 2; ++rw) {
    run<128>(1, rw);
    run<128>(2, rw);
    run<128>(4, rw);
    run<64>(4, rw);
  }
  return 0;
}

// tmem_align.cu — does tcgen05.ld/st.32x32b.x16 accept a column offset that is not a multiple
// of 16 (14-column row slots)?  Writes a pattern with x2 stores, reads it back with x16 at
// column 14 and checks.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k(int* out) {
  __shared__ uint32_t ta;
  const int w = threadIdx.x >> 5;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;\n" ::"r"((uint32_t)__cvta_generic_to_shared(&ta)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t base = ta + ((uint32_t)(w * 32) << 16);
  for (int c = 0; c < 64; c += 2)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};\n" ::"r"(base + c), "r"(c * 1000 + threadIdx.x), "r"((c + 1) * 1000 + threadIdx.x));
  asm volatile("tcgen05.wait::st.sync.aligned;\n");
  uint32_t v[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                 "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
               : "r"(base + 14));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n");
  int bad = 0;
  for (int j = 0; j < 16; ++j) bad += (v[j] != (uint32_t)((14 + j) * 1000 + threadIdx.x));
  atomicAdd(out, bad);
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;\n" ::"r"(ta));
}
int main() {
  int* d; cudaMalloc(&d, 4); cudaMemset(d, 0, 4);
  k<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  int h = -1; cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
  printf("x16 at column 14: %s, mismatches %d\n", cudaGetErrorString(e), h);
  return 0;
}

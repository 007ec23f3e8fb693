// lpb_tmem.cuh — Blackwell tensor memory (TMEM) used as thread-private storage by ordinary
// warps (tcgen05.alloc / ld / st, no MMA): 128 lanes x up to 512 columns of 32 bits per SM.
// Warp w of a CTA reaches TMEM lanes 32(w % 4) .. 32(w % 4) + 31 with the 32x32b shapes, one
// lane per thread, and the column offset is a register operand: a per-thread array with
// dynamic indexing and its own datapath (measured with scripts/ubench/tmem_bw.cu on a B200:
// ≈ 155 B/cycle/SM read plus as much written, 4 CTAs of 4 warps each, load-update-store).
// All tcgen05.ld/st are .sync.aligned: every lane of the warp executes them with the same
// column offset (each lane then reads / writes its own TMEM lane).
#pragma once
#include <cstdint>

#include "lpb_async.cuh"

namespace lpb {

// Warp-wide: allocate NCOL columns (a power of two >= 32) for this CTA, address -> *dst.
template <int NCOL>
__device__ __forceinline__ void tm_alloc(uint32_t* dst) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                   smem_u32(dst)), "n"(NCOL));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
}
// Runtime column count (a power of two >= 32).
__device__ __forceinline__ void tm_alloc_n(uint32_t* dst, uint32_t ncol) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                   smem_u32(dst)), "r"(ncol));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
}
__device__ __forceinline__ void tm_dealloc_n(uint32_t taddr, uint32_t ncol) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncol));
}
template <int NCOL>
__device__ __forceinline__ void tm_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "n"(NCOL));
}
__device__ __forceinline__ void tm_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tm_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// 16 consecutive columns of this thread's lane (8 doubles).
__device__ __forceinline__ void tm_ld16(uint32_t addr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(addr));
}
__device__ __forceinline__ void tm_st16(uint32_t addr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
      ::"r"(addr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]),
        "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]),
        "r"(v[14]), "r"(v[15])
      : "memory");
}
// 8 / 4 consecutive columns (4 / 2 doubles).
__device__ __forceinline__ void tm_ld8(uint32_t addr, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                 "=r"(v[6]), "=r"(v[7])
               : "r"(addr));
}
__device__ __forceinline__ void tm_st8(uint32_t addr, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n"
               ::"r"(addr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]),
                 "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void tm_ld4(uint32_t addr, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(addr));
}
__device__ __forceinline__ void tm_st4(uint32_t addr, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};\n"
               ::"r"(addr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3])
               : "memory");
}
// 14 consecutive columns (7 doubles) as x8 + x4 + x2.
__device__ __forceinline__ void tm_ld2(uint32_t addr, uint32_t& lo, uint32_t& hi);
__device__ __forceinline__ void tm_st2(uint32_t addr, uint32_t lo, uint32_t hi);
__device__ __forceinline__ void tm_ld14(uint32_t addr, uint32_t (&v)[14]) {
  tm_ld8(addr, v);
  tm_ld4(addr + 8, v + 8);
  tm_ld2(addr + 12, v[12], v[13]);
}
__device__ __forceinline__ void tm_st14(uint32_t addr, const uint32_t (&v)[14]) {
  tm_st8(addr, v);
  tm_st4(addr + 8, v + 8);
  tm_st2(addr + 12, v[12], v[13]);
}
// 2 consecutive columns (one double).
__device__ __forceinline__ void tm_ld2(uint32_t addr, uint32_t& lo, uint32_t& hi) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];\n" : "=r"(lo), "=r"(hi) : "r"(addr));
}
__device__ __forceinline__ void tm_st2(uint32_t addr, uint32_t lo, uint32_t hi) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};\n" ::"r"(addr), "r"(lo), "r"(hi)
               : "memory");
}
__device__ __forceinline__ double tm_d(uint32_t lo, uint32_t hi) {
  return __hiloint2double((int)hi, (int)lo);
}
__device__ __forceinline__ void tm_split(double d, uint32_t& lo, uint32_t& hi) {
  lo = (uint32_t)__double2loint(d);
  hi = (uint32_t)__double2hiint(d);
}

}  // namespace lpb

// tcgen05 / TMEM building blocks for the tensor-core MLP (sm_100a).
//
// Operand tiles live in shared memory in the 128-byte-swizzled layout: a
// tile is R rows of 32 fp32 values (128 B per row), 16-byte chunk c of row r
// stored at chunk position c ^ (r & 7), rows contiguous, 1024-byte aligned.
// One buffer serves two MMA views:
//   K-major  (rows = M or N, the 32 values = K): A of the point-major GEMMs
//   MN-major (rows = K, the 32 values = M or N): operands of the
//            parameter-gradient GEMMs, where K runs over points.
// fp32-faithful products use the 3xTF32 split: x = hi + lo with
// hi = x truncated to TF32 (exact in TF32) and lo = x - hi (exact in fp32),
// x*y ~ hi*hi + hi*lo + lo*hi (the dropped lo*lo term is 2^-22 relative).
#pragma once

#include <cstdint>

#include "device_utils.cuh"

namespace vpg {
namespace tc {

// ---- TF32 split --------------------------------------------------------------
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

// byte offset of element (row, col) inside a swizzled 32-column tile
__host__ __device__ __forceinline__ uint32_t sw_off(int row, int col) {
  return (uint32_t)row * 128u + ((((uint32_t)col >> 2) ^ ((uint32_t)row & 7u)) << 4) + (((uint32_t)col & 3u) << 2);
}

// store 4 consecutive columns c0..c0+3 (c0 % 4 == 0) of one row as hi / lo
__device__ __forceinline__ void st_split4(char* hi_tile, char* lo_tile, int row, int c0, float a, float b, float c,
                                          float d) {
  const uint32_t off = sw_off(row, c0);
  const float ha = tf32_hi(a), hb = tf32_hi(b), hc = tf32_hi(c), hd = tf32_hi(d);
  *reinterpret_cast<float4*>(hi_tile + off) = make_float4(ha, hb, hc, hd);
  *reinterpret_cast<float4*>(lo_tile + off) = make_float4(a - ha, b - hb, c - hc, d - hd);
}

// ---- descriptors ---------------------------------------------------------------
// shared-memory matrix descriptor (sm100 layout): start >> 4 [0,14), LBO >> 4
// [16,30), SBO >> 4 [32,46), version 1 [46,48), base offset 0, layout type
// SWIZZLE_128B (= 2) [61,64)
__device__ __forceinline__ uint64_t sdesc(uint32_t smem_addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3fffu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3fffu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3fffu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}

// instruction descriptor, kind::tf32, fp32 accumulate
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int a_mn_major, int b_mn_major) {
  return (1u << 4)                          // D format f32
         | (2u << 7)                        // A tf32
         | (2u << 10)                       // B tf32
         | ((uint32_t)a_mn_major << 15)     // A major
         | ((uint32_t)b_mn_major << 16)     // B major
         | ((uint32_t)(N >> 3) << 17)       // N
         | ((uint32_t)(M >> 4) << 24);      // M
}

// ---- tcgen05 -------------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void fence_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// generic-proxy smem writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_smem_to_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]; issued by ONE thread
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on an mbarrier when all previously issued MMAs of this thread are done
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns: thread i of the warp gets TMEM
// lane (warp's lane quarter base + i), columns [col, col + 16).  The wait is
// inside the same asm statement so no consumer of the registers can be
// scheduled before the data has landed.
#define VPG_R16(b)                                                                                          \
  "=r"(r[b + 0]), "=r"(r[b + 1]), "=r"(r[b + 2]), "=r"(r[b + 3]), "=r"(r[b + 4]), "=r"(r[b + 5]),          \
      "=r"(r[b + 6]), "=r"(r[b + 7]), "=r"(r[b + 8]), "=r"(r[b + 9]), "=r"(r[b + 10]), "=r"(r[b + 11]),    \
      "=r"(r[b + 12]), "=r"(r[b + 13]), "=r"(r[b + 14]), "=r"(r[b + 15])

__device__ __forceinline__ void tmem_ld16_wait(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : VPG_R16(0)
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// two 16-column loads, one wait
__device__ __forceinline__ void tmem_ld2x16_wait(uint32_t ta, uint32_t tb, float (&va)[16], float (&vb)[16]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%32];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, "
      "[%33];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : VPG_R16(0), VPG_R16(16)
      : "r"(ta), "r"(tb)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    va[i] = __uint_as_float(r[i]);
    vb[i] = __uint_as_float(r[16 + i]);
  }
}
#undef VPG_R16

}  // namespace tc
}  // namespace vpg

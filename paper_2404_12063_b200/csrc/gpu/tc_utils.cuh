// tcgen05 / TMEM building blocks for the tensor-core MLP (sm_100a).
//
// fp32-faithful products on the bf16 tensor cores: every operand x is split
// into three bf16 parts x = h + m + l (h = bf16(x), m = bf16(x - h),
// l = bf16(x - h - m), rounded with integer ops; 24+ significant bits in
// total) and a product is the
// sum of the six terms hh + hm + mh + mm + hl + lh (the dropped ml, lm, ll
// terms are below 2^-23 relative), accumulated in fp32 in TMEM.  Six bf16
// MMAs cost the same tensor time as three TF32 ones.
//
// Operand tiles live in shared memory as R rows of 32 bf16 (64 B per row)
// in the 64-byte-swizzled layout (16-byte chunk c of row r stored at chunk
// c ^ ((r >> 1) & 3)), rows contiguous, 8-row atoms of 512 B, 1024-byte
// aligned.  The same tile is a valid operand in both majors:
//   K-major  (rows = M or N, the 32 values = K): point-major GEMM operands
//   MN-major (rows = K, the 32 values = M or N): the parameter-gradient GEMM,
//            whose K runs over points.
// (MN-major TF32 operands would need a different swizzle than K-major ones,
// which is why the split is bf16 and not TF32.)
#pragma once

#include <cuda_bf16.h>

#include <cstdint>

#include "device_utils.cuh"

namespace vpg {
namespace tc {

constexpr int kRowBytes = 64;  // 32 bf16

// byte offset of the 16-byte chunk holding columns [8 chunk, 8 chunk + 8) of row
__host__ __device__ __forceinline__ uint32_t sw_chunk(int row, int chunk) {
  return (uint32_t)row * kRowBytes + ((((uint32_t)chunk) ^ (((uint32_t)row >> 1) & 3u)) << 4);
}

struct Split8 {
  uint4 h, m, l;
};

// x rounded to 8 significant bits (round half away from zero on the
// magnitude), as a float whose low 16 bits are zero, i.e. a bf16 value.
// Integer ops only: the F2F conversion path is a quarter-rate pipe.
__device__ __forceinline__ float bf16_hi(float x) { return __uint_as_float((__float_as_uint(x) + 0x8000u) & 0xffff0000u); }

// two bf16-valued floats -> packed bf16x2 (a in the low half)
__device__ __forceinline__ uint32_t pack2f(float a, float b) {
  return __byte_perm(__float_as_uint(a), __float_as_uint(b), 0x7632);
}

// three-way bf16 split of 8 consecutive values, exact: h = x rounded to 8
// bits, r = x - h (exact, <= 16 significant bits), m = r truncated to 8 bits,
// l = r - m (exact and already 8 bits).  |m| <= 2^-8 |x|, |l| <= 2^-16 |x|,
// so the dropped ml + lm + ll terms are below 2^-23 relative.  Integer and
// FADD ops only (5 per value).
__device__ __forceinline__ Split8 split8(const float* v) {
  uint32_t h[4], m[4], l[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float hf[2], mf[2], lf[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const float x = v[2 * k + e];
      hf[e] = bf16_hi(x);
      const float r = x - hf[e];
      mf[e] = __uint_as_float(__float_as_uint(r) & 0xffff0000u);
      lf[e] = r - mf[e];
    }
    h[k] = pack2f(hf[0], hf[1]);
    m[k] = pack2f(mf[0], mf[1]);
    l[k] = pack2f(lf[0], lf[1]);
  }
  return {make_uint4(h[0], h[1], h[2], h[3]), make_uint4(m[0], m[1], m[2], m[3]), make_uint4(l[0], l[1], l[2], l[3])};
}

// store 8 consecutive columns [8 chunk, +8) of one row into the three part
// tiles at base, base + part_stride, base + 2 part_stride
__device__ __forceinline__ void st_split8(char* base, uint32_t part_stride, int row, int chunk, const float* v) {
  const Split8 s = split8(v);
  const uint32_t off = sw_chunk(row, chunk);
  *reinterpret_cast<uint4*>(base + off) = s.h;
  *reinterpret_cast<uint4*>(base + part_stride + off) = s.m;
  *reinterpret_cast<uint4*>(base + 2 * part_stride + off) = s.l;
}

__device__ __forceinline__ void unpack8(uint4 q, float* v) {
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    v[2 * k] = __uint_as_float(w[k] << 16);
    v[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
  }
}

// read back 8 columns as h + m + l
__device__ __forceinline__ void ld_join8(const char* base, uint32_t part_stride, int row, int chunk, float* v) {
  const uint32_t off = sw_chunk(row, chunk);
  float h[8], m[8], l[8];
  unpack8(*reinterpret_cast<const uint4*>(base + off), h);
  unpack8(*reinterpret_cast<const uint4*>(base + part_stride + off), m);
  unpack8(*reinterpret_cast<const uint4*>(base + 2 * part_stride + off), l);
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = h[k] + (m[k] + l[k]);
}

// ---- fp16 two-part split (tc2_step_kernel.cuh) ------------------------------
// y = s * x with a power-of-two s (exact), h = f16(y), l = f16(y - h): y - h
// is exact in fp32 and h + l carries 22 significant bits, so the three
// products hh' + hl' + lh' are fp32-faithful (dropped ll' < 2^-22 relative)
// as long as s keeps |y| inside the fp16 normal range (the caller scales by
// a bound, see tc2_step_kernel.cuh).  cvt.rn.f16x2.f32 runs on the ALU pipe
// (measured 2 warp-instr/clk/SM on B200, the LOP3 rate).
__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ float f16lo(uint32_t w) {
  float f;
  asm("{\n .reg .b16 lo, hi;\n mov.b32 {lo, hi}, %1;\n cvt.f32.f16 %0, lo;\n}" : "=f"(f) : "r"(w));
  return f;
}
__device__ __forceinline__ float f16hi(uint32_t w) {
  float f;
  asm("{\n .reg .b16 lo, hi;\n mov.b32 {lo, hi}, %1;\n cvt.f32.f16 %0, hi;\n}" : "=f"(f) : "r"(w));
  return f;
}
// y - h for both halves of a packed pair: one mixed-precision FMA per value
// (fma.rn.f32.f16, y + h * -1: a single FHFMA reading the half in place, no
// f16 -> f32 unpack); exact, since y - h is representable in fp32
__device__ __forceinline__ float2 rem_f16x2(uint32_t h, float2 y) {
  float2 r;
  asm("{\n .reg .b16 lo, hi, m1;\n mov.b16 m1, 0xBC00;\n mov.b32 {lo, hi}, %2;\n"
      " fma.rn.f32.f16 %0, lo, m1, %3;\n fma.rn.f32.f16 %1, hi, m1, %4;\n}"
      : "=f"(r.x), "=f"(r.y) : "r"(h), "f"(y.x), "f"(y.y));
  return r;
}
// h + l of a packed pair in fp32 (round to nearest, as float(h) + float(l)):
// the l halves unpacked, then one mixed-precision add each reading h in place
__device__ __forceinline__ float2 join_f16x2(uint32_t h, uint32_t l) {
  float2 v;
  asm("{\n .reg .b16 hl, hh, ll, lh;\n .reg .f32 t0, t1;\n mov.b32 {hl, hh}, %2;\n mov.b32 {ll, lh}, %3;\n"
      " cvt.f32.f16 t0, ll;\n cvt.f32.f16 t1, lh;\n add.rn.f32.f16 %0, hl, t0;\n add.rn.f32.f16 %1, hh, t1;\n}"
      : "=f"(v.x), "=f"(v.y) : "r"(h), "r"(l));
  return v;
}
// store 8 consecutive columns [8 chunk, +8) of one row, scaled by s, into
// the two part tiles at base (h) and base + part_stride (l)
__device__ __forceinline__ void st_split8_h(char* base, uint32_t part_stride, int row, int chunk, const float* v,
                                            float s) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float y0 = v[2 * k] * s, y1 = v[2 * k + 1] * s;
    h[k] = pack_f16x2(y0, y1);
    const float2 r = rem_f16x2(h[k], make_float2(y0, y1));
    l[k] = pack_f16x2(r.x, r.y);
  }
  const uint32_t off = sw_chunk(row, chunk);
  *reinterpret_cast<uint4*>(base + off) = make_uint4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<uint4*>(base + part_stride + off) = make_uint4(l[0], l[1], l[2], l[3]);
}
// the same with a precomputed swizzled byte offset; SCALE = false skips the
// multiply (values already scaled)
template <bool SCALE>
__device__ __forceinline__ void st_split8_ho(char* base, uint32_t part_stride, uint32_t off, const float* v, float s) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 y = SCALE ? __fmul2_rn(make_float2(v[2 * k], v[2 * k + 1]), make_float2(s, s))
                           : make_float2(v[2 * k], v[2 * k + 1]);
    h[k] = pack_f16x2(y.x, y.y);
    const float2 r = rem_f16x2(h[k], y);
    l[k] = pack_f16x2(r.x, r.y);
  }
  *reinterpret_cast<uint4*>(base + off) = make_uint4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<uint4*>(base + part_stride + off) = make_uint4(l[0], l[1], l[2], l[3]);
}
template <bool UNSCALE>
__device__ __forceinline__ void ld_join8_ho(const char* base, uint32_t part_stride, uint32_t off, float inv_s,
                                            float* v) {
  const uint4 h = *reinterpret_cast<const uint4*>(base + off);
  const uint4 l = *reinterpret_cast<const uint4*>(base + part_stride + off);
  const uint32_t hw[4] = {h.x, h.y, h.z, h.w}, lw[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float2 a = join_f16x2(hw[k], lw[k]);
    if (UNSCALE) a = __fmul2_rn(a, make_float2(inv_s, inv_s));
    v[2 * k] = a.x;
    v[2 * k + 1] = a.y;
  }
}
// read back 8 columns as (h + l) * inv_s
__device__ __forceinline__ void ld_join8_h(const char* base, uint32_t part_stride, int row, int chunk, float inv_s,
                                           float* v) {
  const uint32_t off = sw_chunk(row, chunk);
  const uint4 h = *reinterpret_cast<const uint4*>(base + off);
  const uint4 l = *reinterpret_cast<const uint4*>(base + part_stride + off);
  const uint32_t hw[4] = {h.x, h.y, h.z, h.w}, lw[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 a = join_f16x2(hw[k], lw[k]);
    v[2 * k] = a.x * inv_s;
    v[2 * k + 1] = a.y * inv_s;
  }
}
// 2^k as a float, k clamped to the normal range
__device__ __forceinline__ float exp2i(int k) {
  k = max(-126, min(127, k));
  return __uint_as_float((uint32_t)(127 + k) << 23);
}
// the exponent e with b < 2^e for a positive normal b (-1000 for zero,
// denormal or NaN: "no bound"); inf gives 129
__device__ __forceinline__ int bound_exp(float b) {
  const uint32_t bits = __float_as_uint(b);
  const int E = (int)((bits >> 23) & 0xffu);
  if (!(b > 0.f) || E == 0) return -1000;
  return E - 126;
}

// the six bf16x3 part products (a part, b part), smallest first (probe mode 3)
__device__ constexpr int kProdA[6] = {2, 0, 1, 1, 0, 0};
__device__ constexpr int kProdB[6] = {0, 2, 1, 0, 1, 0};

// ---- descriptors ---------------------------------------------------------------
// shared-memory matrix descriptor (sm100): start >> 4 [0,14), LBO >> 4
// [16,30), SBO >> 4 [32,46), version 1 [46,48), base offset 0, layout type
// SWIZZLE_64B (= 4) [61,64)
__device__ __forceinline__ uint64_t sdesc(uint32_t smem_addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3fffu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3fffu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3fffu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)4u << 61;
  return d;
}
// K-major operand: rows = M/N at 64 B, 8-row groups 512 B apart; K step of
// 16 bf16 = +32 B inside the row
__device__ __forceinline__ uint64_t kdesc(uint32_t smem_addr) { return sdesc(smem_addr, 16, 512); }
// MN-major operand: rows = K, MN blocks of 32 at lbo; K step of 16 rows = +1024 B
__device__ __forceinline__ uint64_t mndesc(uint32_t smem_addr, uint32_t lbo) { return sdesc(smem_addr, lbo, 512); }

// instruction descriptor, kind::f16 with bf16 inputs, fp32 accumulate
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn_major, int b_mn_major) {
  return (1u << 4)                       // D format f32
         | (1u << 7)                     // A bf16
         | (1u << 10)                    // B bf16
         | ((uint32_t)a_mn_major << 15)  // A major
         | ((uint32_t)b_mn_major << 16)  // B major
         | ((uint32_t)(N >> 3) << 17)    // N
         | ((uint32_t)(M >> 4) << 24);   // M
}

// instruction descriptor, kind::f16 with fp16 inputs, fp32 accumulate
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N, int a_mn_major, int b_mn_major) {
  return (1u << 4) | ((uint32_t)a_mn_major << 15) | ((uint32_t)b_mn_major << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
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
// true on one lane of the (converged) warp
__device__ __forceinline__ bool elect_one() {
  uint32_t e;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(e));
  return e != 0;
}
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// warp-collective forms: called by all 32 threads of ONE converged warp, one
// elected lane issues (no divergent single-thread branch around the MMA, so
// the descriptors stay warp-uniform and no elect loop is generated)
__device__ __forceinline__ void mma_warp(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
template <int S>
__device__ __forceinline__ void mma_warp_sd(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc) {
  static_assert(S >= 0 && S <= 15, "scale-input-d range");
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, 1, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p, %4;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "n"(S)
      : "memory");
}
// out of line: the 16-way switch is the rare path (a tile whose product
// scale drops below the accumulated one), kept out of the hot code's I-cache
#ifndef VPG_SD_NOINLINE
#define VPG_SD_NOINLINE 1
#endif
#if VPG_SD_NOINLINE
static __device__ __noinline__
#else
__device__ __forceinline__
#endif
void mma_warp_sd(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, int s) {
  switch (s) {
#define VPG_SDW(k) \
  case k:          \
    mma_warp_sd<k>(d, a, b, idesc); \
    break;
    VPG_SDW(0) VPG_SDW(1) VPG_SDW(2) VPG_SDW(3) VPG_SDW(4) VPG_SDW(5) VPG_SDW(6) VPG_SDW(7)
    VPG_SDW(8) VPG_SDW(9) VPG_SDW(10) VPG_SDW(11) VPG_SDW(12) VPG_SDW(13) VPG_SDW(14) default: mma_warp_sd<15>(d, a, b, idesc);
#undef VPG_SDW
  }
}
__device__ __forceinline__ void commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(bar))
      : "memory");
}

// D[tmem] = A * B + D * 2^-S (scale-input-d, kind::f16): accumulates onto a
// scaled-down accumulator, S in [0, 15]
template <int S>
__device__ __forceinline__ void mma_f16_sd(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc) {
  static_assert(S >= 0 && S <= 15, "scale-input-d range");
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, 1, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p, %4;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "n"(S)
      : "memory");
}
// runtime S in [0, 15]
__device__ __forceinline__ void mma_f16_sd(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, int s) {
  switch (s) {
#define VPG_SD(k) \
  case k:         \
    mma_f16_sd<k>(d, a, b, idesc); \
    break;
    VPG_SD(0) VPG_SD(1) VPG_SD(2) VPG_SD(3) VPG_SD(4) VPG_SD(5) VPG_SD(6) VPG_SD(7)
    VPG_SD(8) VPG_SD(9) VPG_SD(10) VPG_SD(11) VPG_SD(12) VPG_SD(13) VPG_SD(14) default: mma_f16_sd<15>(d, a, b, idesc);
#undef VPG_SD
  }
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
#define VPG_LD16 "tcgen05.ld.sync.aligned.32x32b.x16.b32 "

// three 16-column loads, one wait
__device__ __forceinline__ void tmem_ld3x16_wait(uint32_t ta, uint32_t tb, uint32_t tc_, float (&va)[16],
                                                 float (&vb)[16], float (&vc)[16]) {
  uint32_t r[48];
  asm volatile(VPG_LD16 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%48];\n\t" VPG_LD16
                        "{%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%49];\n\t" VPG_LD16
                        "{%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47}, [%50];\n\t"
                        "tcgen05.wait::ld.sync.aligned;"
               : VPG_R16(0), VPG_R16(16), VPG_R16(32)
               : "r"(ta), "r"(tb), "r"(tc_)
               : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    va[i] = __uint_as_float(r[i]);
    vb[i] = __uint_as_float(r[16 + i]);
    vc[i] = __uint_as_float(r[32 + i]);
  }
}
#define VPG_R8(b)                                                                                           \
  "=r"(r[b + 0]), "=r"(r[b + 1]), "=r"(r[b + 2]), "=r"(r[b + 3]), "=r"(r[b + 4]), "=r"(r[b + 5]),          \
      "=r"(r[b + 6]), "=r"(r[b + 7])
#define VPG_LD8 "tcgen05.ld.sync.aligned.32x32b.x8.b32 "
// three 8-column loads, one wait
__device__ __forceinline__ void tmem_ld3x8_wait(uint32_t ta, uint32_t tb, uint32_t tc_, float (&va)[8],
                                                float (&vb)[8], float (&vc)[8]) {
  uint32_t r[24];
  asm volatile(VPG_LD8 "{%0,%1,%2,%3,%4,%5,%6,%7}, [%24];\n\t" VPG_LD8
                       "{%8,%9,%10,%11,%12,%13,%14,%15}, [%25];\n\t" VPG_LD8
                       "{%16,%17,%18,%19,%20,%21,%22,%23}, [%26];\n\t"
                       "tcgen05.wait::ld.sync.aligned;"
               : VPG_R8(0), VPG_R8(8), VPG_R8(16)
               : "r"(ta), "r"(tb), "r"(tc_)
               : "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    va[i] = __uint_as_float(r[i]);
    vb[i] = __uint_as_float(r[8 + i]);
    vc[i] = __uint_as_float(r[16 + i]);
  }
}
// one 16-column load
__device__ __forceinline__ void tmem_ld1x16_wait(uint32_t ta, float (&va)[16]) {
  uint32_t r[16];
  asm volatile(VPG_LD16 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
                        "tcgen05.wait::ld.sync.aligned;"
               : VPG_R16(0)
               : "r"(ta)
               : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) va[i] = __uint_as_float(r[i]);
}
// one / two 8-column loads, one wait
__device__ __forceinline__ void tmem_ld1x8_wait(uint32_t ta, float (&va)[8]) {
  uint32_t r[8];
  asm volatile(VPG_LD8 "{%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t"
                       "tcgen05.wait::ld.sync.aligned;"
               : VPG_R8(0)
               : "r"(ta)
               : "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) va[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld2x8_wait(uint32_t ta, uint32_t tb, float (&va)[8], float (&vb)[8]) {
  uint32_t r[16];
  asm volatile(VPG_LD8 "{%0,%1,%2,%3,%4,%5,%6,%7}, [%16];\n\t" VPG_LD8
                       "{%8,%9,%10,%11,%12,%13,%14,%15}, [%17];\n\t"
                       "tcgen05.wait::ld.sync.aligned;"
               : VPG_R8(0), VPG_R8(8)
               : "r"(ta), "r"(tb)
               : "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    va[i] = __uint_as_float(r[i]);
    vb[i] = __uint_as_float(r[8 + i]);
  }
}
// store 8 consecutive columns of this warp's lane quarter (thread i: lane
// base + i), then wait for the store to complete
__device__ __forceinline__ void tmem_st1x8_wait(uint32_t ta, const float (&v)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n\t"
      "tcgen05.wait::st.sync.aligned;" ::"r"(ta),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
      : "memory");
}
// N in {8, 16} columns per load
template <int N>
__device__ __forceinline__ void tmem_ld3_wait(uint32_t ta, uint32_t tb, uint32_t tc_, float (&va)[N], float (&vb)[N],
                                              float (&vc)[N]) {
  if constexpr (N == 16)
    tmem_ld3x16_wait(ta, tb, tc_, va, vb, vc);
  else
    tmem_ld3x8_wait(ta, tb, tc_, va, vb, vc);
}
#undef VPG_LD8
#undef VPG_R8
#undef VPG_LD16
#undef VPG_R16

}  // namespace tc
}  // namespace vpg

// Small sm_100a device helpers: vector shared-memory access, mbarrier and
// bulk-copy (TMA 1-D, cp.async.bulk) primitives, exact activations.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace vpg {

constexpr int kThreads = 128;  // threads per CTA of the step kernels
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ float4 lds4(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}
__device__ __forceinline__ void sts4(float* p, float4 v) {
  *reinterpret_cast<float4*>(p) = v;
}

// ---- mbarrier + cp.async.bulk (1-D TMA) ------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
      "[%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
#ifndef VPG_MBAR_HINT
#define VPG_MBAR_HINT 1
#endif
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
#if VPG_MBAR_HINT
  // with a suspend-time hint the warp sleeps until the phase completes (or
  // the hint expires) instead of spinning on issue slots other warps need
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(0x989680u)
      : "memory");
#else
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
#endif
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// ---- programmatic dependent launch (PDL) -----------------------------------
// A kernel launched with the programmatic-stream-serialization attribute may
// be scheduled while its predecessor still runs; pdl_wait() blocks until the
// predecessor grid has completed and its writes are visible (a no-op for a
// normal launch), pdl_trigger() lets this kernel's successor be scheduled
// early.  Called first thing, before any read of predecessor data.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---- activations (ActDerivs, network.hpp:171-192, from the OUTPUT z) --------
// s1 = act', kap = act''/act' so that s2 = kap * s1:
//   tanh:    s1 = 1 - z^2,   kap = -2 z
//   sigmoid: s1 = z (1 - z), kap = 1 - 2 z
// Branch-free, compact evaluations (the step kernel inlines ~100 of them, so
// code size matters as much as latency):
//   tanh |x| <  0.4 : x + x^3 P(x^2), degree-4 minimax, <= 0.63 ulp
//   tanh |x| >= 0.4 : 1 - 2 / (2^(2|x| log2 e) + 1) with MUFU ex2/rcp and one
//                     Newton step; the ex2 error is attenuated by
//                     2e/(e^2-1) <= 1.13 at the switch point
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_newton(float d) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d));
  return fmaf(r, fmaf(-d, r, 1.0f), r);  // one Newton step
}

// ---- packed fp32x2 (FFMA2 / FMUL2 / FADD2, sm_100): two lanes of work per
// issued instruction at the same FMA throughput, i.e. half the issue slots
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 f2s(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }

#ifndef VPG_TANH2_NEWTON
#define VPG_TANH2_NEWTON 0  // packed tanh: Newton step on rcp.approx (off: |x| >= 0.4 branch within ~2 ulp; parity suite unchanged)
#endif

constexpr int kActTanh = 0;
constexpr int kActSigmoid = 1;

template <int ACT>
struct Act;

template <>
struct Act<kActTanh> {
  static __device__ __forceinline__ float value(float x) {
    const float ax = fabsf(x);
    const float x2 = x * x;
    float p = -0.007364633358913433f;
    p = fmaf(p, x2, 0.021618979731563185f);
    p = fmaf(p, x2, -0.05394892778111454f);
    p = fmaf(p, x2, 0.1333326813390213f);
    p = fmaf(p, x2, -0.3333333262496359f);
    const float small = fmaf(x * x2, p, x);
    // |x| >= 9.1 rounds to 1.0f (as the correctly rounded tanh does); the
    // clamp at 15 keeps e finite for the Newton step
    const float e = ex2_approx(fminf(ax, 15.0f) * 2.8853900817779268f);
    const float big = fmaf(-2.0f, rcp_newton(e + 1.0f), 1.0f);
    return ax < 0.4f ? small : copysignf(big, x);
  }
  static __device__ __forceinline__ float s1(float z) { return fmaf(-z, z, 1.0f); }
  static __device__ __forceinline__ float kap(float z) { return -2.0f * z; }
  // two values at once, the same operations as value() in packed fp32x2
  static __device__ __forceinline__ float2 value2(float2 x) {
    const float2 x2 = __fmul2_rn(x, x);
    float2 p = __ffma2_rn(f2s(-0.007364633358913433f), x2, f2s(0.021618979731563185f));
    p = __ffma2_rn(p, x2, f2s(-0.05394892778111454f));
    p = __ffma2_rn(p, x2, f2s(0.1333326813390213f));
    p = __ffma2_rn(p, x2, f2s(-0.3333333262496359f));
    const float2 small = __ffma2_rn(__fmul2_rn(x, x2), p, x);
    const float2 ax = f2(fabsf(x.x), fabsf(x.y));
    const float2 t = __fmul2_rn(f2(fminf(ax.x, 15.0f), fminf(ax.y, 15.0f)), f2s(2.8853900817779268f));
    const float2 d = __fadd2_rn(f2(ex2_approx(t.x), ex2_approx(t.y)), f2s(1.0f));
    float2 r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r.x) : "f"(d.x));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r.y) : "f"(d.y));
#if VPG_TANH2_NEWTON
    r = __ffma2_rn(r, __ffma2_rn(f2(-d.x, -d.y), r, f2s(1.0f)), r);  // one Newton step
#endif
    const float2 big = __ffma2_rn(f2s(-2.0f), r, f2s(1.0f));
    return f2(ax.x < 0.4f ? small.x : copysignf(big.x, x.x), ax.y < 0.4f ? small.y : copysignf(big.y, x.y));
  }
  static __device__ __forceinline__ float2 s1_2(float2 z) { return __ffma2_rn(f2(-z.x, -z.y), z, f2s(1.0f)); }
  static __device__ __forceinline__ float2 kap2(float2 z) { return __fmul2_rn(f2s(-2.0f), z); }
  // kap is -2 z: callers may fold the -2 into a scalar factor (exact)
  static constexpr bool kKapLinear = true;
};

template <>
struct Act<kActSigmoid> {
  static __device__ __forceinline__ float value(float x) {
    // 1 / (1 + exp(-x)); exp via ex2 (rel. err ~2^-22), overflow -> 0
    const float e = ex2_approx(fminf(-x * 1.4426950408889634f, 126.0f));
    return rcp_newton(1.0f + e);
  }
  static __device__ __forceinline__ float s1(float z) { return z * (1.0f - z); }
  static __device__ __forceinline__ float kap(float z) { return 1.0f - 2.0f * z; }
  static __device__ __forceinline__ float2 value2(float2 x) { return f2(value(x.x), value(x.y)); }
  static __device__ __forceinline__ float2 s1_2(float2 z) { return __fmul2_rn(z, __fadd2_rn(f2s(1.0f), f2(-z.x, -z.y))); }
  static __device__ __forceinline__ float2 kap2(float2 z) { return __ffma2_rn(f2s(-2.0f), z, f2s(1.0f)); }
  static constexpr bool kKapLinear = false;
};

// network.hpp:130-138
__device__ __forceinline__ float softplusf(float x) {
  return log1pf(expf(-fabsf(x))) + fmaxf(x, 0.0f);
}
__device__ __forceinline__ float sigmoidf(float x) { return 1.0f / (1.0f + expf(-x)); }

__device__ __forceinline__ bool finitef(float x) { return isfinite(x); }

}  // namespace vpg

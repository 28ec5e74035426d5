// Kernel-variant registry shared by the per-variant translation units (each
// instantiates the step kernels for one hidden shape, compiled in parallel).
#pragma once

#include <cstddef>
#include <vector>

#include "step_kernel.cuh"

namespace vpg {

using StepFn = void (*)(StepArgs);

struct Variant {
  int H, D, C;
  StepFn fused, forward, reverse;
  int off_union;  // floats before the union
  int rev_need;   // floats the reverse phase needs in the union
  size_t (*smem)(int, int);
};

#define VPG_VARIANTS(X) \
  X(30, 3, 1) X(30, 3, 2) X(20, 2, 1) X(20, 2, 2) X(50, 3, 1) X(16, 1, 1) X(16, 1, 2) X(16, 2, 1)

#define VPG_DECL(H, D, C) Variant variant_##H##_##D##_##C();
VPG_VARIANTS(VPG_DECL)
#undef VPG_DECL

#ifdef VPG_DEFINE_VARIANT
template <int H, int D, int C>
Variant make_variant() {
  using LY = Layout<H, D, C>;
  Variant v;
  v.H = H;
  v.D = D;
  v.C = C;
  v.fused = step_kernel<H, D, C, kModeFused>;
  v.forward = step_kernel<H, D, C, kModeForward>;
  v.reverse = step_kernel<H, D, C, kModeReverse>;
  v.off_union = LY::OFF_UNION;
  v.rev_need = LY::REV_NEED;
  v.smem = [](int u, int r) { return step_smem_bytes<H, D, C>(u, r); };
  return v;
}
#define VPG_DEFINE(H, D, C) \
  Variant variant_##H##_##D##_##C() { return make_variant<H, D, C>(); }
#endif

}  // namespace vpg

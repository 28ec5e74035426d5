// Kernel-variant registry shared by the per-variant translation units (each
// instantiates the step kernels for one hidden shape, compiled in parallel).
#pragma once

#include <cstddef>
#include <vector>

#include "step_kernel.cuh"

namespace vpg {

using StepFn = void (*)(StepArgs);

struct Variant {
  int H, D, C, ACT;
  StepFn fused, forward, reverse;  // CUDA-core step (step_kernel.cuh): every shape
  StepFn tc2;      // tensor-core step (tc2_step_kernel.cuh), nullptr if the shape has none
  StepFn tc2_fwd;  // its forward-only / reverse-only modes (split path, evaluate)
  StepFn tc2_rev;
  StepFn tc2_lat;       // the fused step with 8 units per thread (512 threads): grids of <= 1 tile per SM
  size_t tc2_lat_smem;
  int tc2_lat_nt;
  size_t tc2_smem;
  int tc2_nt;        // threads per CTA
  int tc2_mp;        // points per tile
  int tc2_buf;       // bytes of one operand buffer (the slab aliases buffer A)
  int tc2_scratch;   // floats of the per-CTA spill scratch per MMA layer
  int off_union;  // floats before the union
  int rev_need;   // floats the reverse phase needs in the union
  size_t (*smem)(int, int);
};

// (hidden width, hidden layers, output channels, activation 0 tanh / 1 sigmoid);
// a network uses the narrowest instantiated width >= its widest hidden layer,
// narrower layers zero-padded exactly.  Served (reference networks are
// [2, hidden..., n_out], config.hpp:429-434):
//   1-2 hidden layers, width <= 64, 1 or 2 outputs;
//   3 hidden layers, width <= 62 with one output (tensor cores), <= 50 with two;
//   4 hidden layers, width <= 36 (CUDA cores: the per-point state of wider
//   nets exceeds shared memory);
// tanh or sigmoid everywhere.  Tensor-core step (tc2) for 2-3 hidden layers of
// width <= 62, one output or two (the spatial-eps head); the CUDA-core step
// for everything else.
#define VPG_VARIANTS(X) \
  X(30, 1, 1, 0) X(30, 1, 1, 1) X(30, 1, 2, 0) X(30, 1, 2, 1) X(64, 1, 1, 0) X(64, 1, 1, 1) \
  X(64, 1, 2, 0) X(64, 1, 2, 1) X(30, 2, 1, 0) X(30, 2, 1, 1) X(62, 2, 1, 0) X(62, 2, 1, 1) \
  X(64, 2, 1, 0) X(64, 2, 1, 1) X(30, 2, 2, 0) X(30, 2, 2, 1) X(64, 2, 2, 0) X(64, 2, 2, 1) \
  X(30, 3, 1, 0) X(30, 3, 1, 1) X(50, 3, 1, 0) X(50, 3, 1, 1) X(62, 3, 1, 0) X(62, 3, 1, 1) \
  X(30, 3, 2, 0) X(30, 3, 2, 1) X(50, 3, 2, 0) X(50, 3, 2, 1) X(36, 4, 1, 0) X(36, 4, 1, 1) \
  X(36, 4, 2, 0) X(36, 4, 2, 1)

#define VPG_DECL(H, D, C, A) Variant variant_##H##_##D##_##C##_##A();
VPG_VARIANTS(VPG_DECL)
#undef VPG_DECL

#ifdef VPG_DEFINE_VARIANT
}  // namespace vpg
#include "tc2_step_kernel.cuh"
namespace vpg {
template <int H, int D, int C, int A>
Variant make_variant() {
  using LY = Layout<H, D, C>;
  Variant v{};
  v.H = H;
  v.D = D;
  v.C = C;
  v.ACT = A;
  v.fused = step_kernel<H, D, C, A, kModeFused>;
  v.forward = step_kernel<H, D, C, A, kModeForward>;
  v.reverse = step_kernel<H, D, C, A, kModeReverse>;
  v.off_union = LY::OFF_UNION;
  v.rev_need = LY::REV_NEED;
  v.smem = [](int u, int r) { return step_smem_bytes<H, D, C>(u, r); };
  if constexpr ((D == 2 || D == 3) && H <= 63) {
    if constexpr (tc2_step_smem_bytes<H, D, C>() <= 227 * 1024) {
    using CF = t2::Cfg<H>;
    v.tc2 = tc2_step_kernel<H, D, A, kModeFused, C>;
    v.tc2_fwd = tc2_step_kernel<H, D, A, kModeForward, C>;
    v.tc2_rev = tc2_step_kernel<H, D, A, kModeReverse, C>;
    v.tc2_smem = tc2_step_smem_bytes<H, D, C>();
    v.tc2_nt = CF::NT;
    v.tc2_mp = CF::MP;
    v.tc2_buf = CF::kBuf;
    v.tc2_scratch = CF::kScratch;
    if constexpr (CF::NB == 1) {
      v.tc2_lat = tc2_step_kernel<H, D, A, kModeFused, C, 8>;
      v.tc2_lat_smem = tc2_step_smem_bytes<H, D, C, 8>();
      v.tc2_lat_nt = t2::Cfg<H, 8>::NT;
    }
    }
  }
  return v;
}
#define VPG_DEFINE(H, D, C, A) \
  Variant variant_##H##_##D##_##C##_##A() { return make_variant<H, D, C, A>(); }
#endif

}  // namespace vpg

// Host view of the strong-form step kernels (sf_step.cu).
#pragma once

#include <cstddef>

#include "step_kernel.cuh"

namespace vpg {

struct SfKernels {
  void (*fused)(StepArgs);    // loss + gradient parts (kModeFused)
  void (*forward)(StepArgs);  // order-2 evaluate (kModeForward)
};
// D hidden layers (1..4), act 0 tanh / 1 sigmoid; {nullptr, nullptr} otherwise
SfKernels sf_kernels(int D, int act);
size_t sf_smem_bytes(int D, int warps);
constexpr int kSfMaxWarps = 8;

}  // namespace vpg

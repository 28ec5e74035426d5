// Host view of the strong-form step kernels (sf_step.cu).
#pragma once

#include <cstddef>

#include "step_kernel.cuh"

namespace vpg {

struct SfKernels {
  void (*fused)(StepArgs);    // loss + gradient parts (kModeFused), warp-tiled mma.sync
  void (*forward)(StepArgs);  // order-2 evaluate (kModeForward)
  // the tcgen05 version (sf2_step_kernel.cuh): 2-3 hidden layers of width
  // <= 31; nullptr otherwise
  void (*tc_fused)(StepArgs);
  void (*tc_forward)(StepArgs);
  size_t tc_smem;
};
constexpr int kSf2Threads = 256, kSf2Points = 128;
// D hidden layers (1..4), act 0 tanh / 1 sigmoid; {nullptr, nullptr} otherwise
SfKernels sf_kernels(int D, int act);
size_t sf_smem_bytes(int D, int warps);
constexpr int kSfMaxWarps = 8;

}  // namespace vpg

// Strong-form step kernels (sf_step_kernel.cuh) for 1-4 hidden layers of
// width <= 32, tanh / sigmoid.
#include "sf2_step_kernel.cuh"
#include "sf_step.h"
#include "sf_step_kernel.cuh"

namespace vpg {

namespace {
template <int D, int A>
SfKernels make() {
  if constexpr (D == 2 || D == 3)
    return {sf_step_kernel<D, A, kModeFused>, sf_step_kernel<D, A, kModeForward>, sf2_step_kernel<31, D, A, kModeFused>,
            sf2_step_kernel<31, D, A, kModeForward>, sf2_step_smem_bytes<D>()};
  else
    return {sf_step_kernel<D, A, kModeFused>, sf_step_kernel<D, A, kModeForward>, nullptr, nullptr, 0};
}
}  // namespace

SfKernels sf_kernels(int D, int act) {
  const int a = act ? 1 : 0;
  switch (D * 2 + a) {
    case 2: return make<1, 0>();
    case 3: return make<1, 1>();
    case 4: return make<2, 0>();
    case 5: return make<2, 1>();
    case 6: return make<3, 0>();
    case 7: return make<3, 1>();
    case 8: return make<4, 0>();
    case 9: return make<4, 1>();
    default: return {nullptr, nullptr, nullptr, nullptr, 0};
  }
}

size_t sf_smem_bytes(int D, int warps) { return sf::smem_bytes(D, warps); }

}  // namespace vpg

// step kernels instantiated for hidden width 36, 4 hidden layer(s), 1 output channel(s), tanh
#define VPG_DEFINE_VARIANT
#include "variant.h"
namespace vpg {
VPG_DEFINE(36, 4, 1, 0)
}  // namespace vpg

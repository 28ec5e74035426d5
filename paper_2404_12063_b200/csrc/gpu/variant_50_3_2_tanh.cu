// step kernels instantiated for hidden width 50, 3 hidden layer(s), 2 output channel(s), tanh
#define VPG_DEFINE_VARIANT
#include "variant.h"
namespace vpg {
VPG_DEFINE(50, 3, 2, 0)
}  // namespace vpg

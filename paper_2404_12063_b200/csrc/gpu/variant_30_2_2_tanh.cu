// step kernels instantiated for hidden width 30, 2 hidden layer(s), 2 output channel(s), tanh
#define VPG_DEFINE_VARIANT
#include "variant.h"
namespace vpg {
VPG_DEFINE(30, 2, 2, 0)
}  // namespace vpg

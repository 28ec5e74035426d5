// step kernels instantiated for hidden width 62, 2 hidden layer(s), 1 output channel(s), tanh
#define VPG_DEFINE_VARIANT
#include "variant.h"
namespace vpg {
VPG_DEFINE(62, 2, 1, 0)
}  // namespace vpg

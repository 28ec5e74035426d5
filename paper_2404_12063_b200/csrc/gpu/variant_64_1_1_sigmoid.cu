// step kernels instantiated for hidden width 64, 1 hidden layer(s), 1 output channel(s), sigmoid
#define VPG_DEFINE_VARIANT
#include "variant.h"
namespace vpg {
VPG_DEFINE(64, 1, 1, 1)
}  // namespace vpg

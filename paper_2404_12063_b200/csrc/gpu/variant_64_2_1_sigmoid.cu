// step kernels instantiated for hidden width 64, 2 hidden layer(s), 1 output channel(s), sigmoid
#define VPG_DEFINE_VARIANT
#include "variant.h"
namespace vpg {
VPG_DEFINE(64, 2, 1, 1)
}  // namespace vpg

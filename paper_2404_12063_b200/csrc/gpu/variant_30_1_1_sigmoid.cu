// step kernels instantiated for hidden width 30, 1 hidden layer(s), 1 output channel(s), sigmoid
#define VPG_DEFINE_VARIANT
#include "variant.h"
namespace vpg {
VPG_DEFINE(30, 1, 1, 1)
}  // namespace vpg

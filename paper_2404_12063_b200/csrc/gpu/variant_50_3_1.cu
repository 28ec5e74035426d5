// step kernels instantiated for hidden width 50, 3 hidden layers, 1 output channel(s)
#define VPG_DEFINE_VARIANT
#include "variant.h"
namespace vpg {
VPG_DEFINE(50, 3, 1)
}  // namespace vpg

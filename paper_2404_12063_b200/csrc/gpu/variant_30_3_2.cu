// step kernels instantiated for hidden width 30, 3 hidden layers, 2 output channel(s)
#define VPG_DEFINE_VARIANT
#include "variant.h"
namespace vpg {
VPG_DEFINE(30, 3, 2)
}  // namespace vpg

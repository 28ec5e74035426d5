// step kernels instantiated for hidden width 20, 2 hidden layers, 2 output channel(s)
#define VPG_DEFINE_VARIANT
#include "variant.h"
namespace vpg {
VPG_DEFINE(20, 2, 2)
}  // namespace vpg

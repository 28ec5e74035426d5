// step kernels instantiated for hidden width 20, 2 hidden layers, 1 output channel(s)
#define VPG_DEFINE_VARIANT
#include "variant.h"
namespace vpg {
VPG_DEFINE(20, 2, 1)
}  // namespace vpg

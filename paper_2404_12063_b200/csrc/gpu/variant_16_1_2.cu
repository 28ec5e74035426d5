// step kernels instantiated for hidden width 16, 1 hidden layers, 2 output channel(s)
#define VPG_DEFINE_VARIANT
#include "variant.h"
namespace vpg {
VPG_DEFINE(16, 1, 2)
}  // namespace vpg

// step kernels instantiated for hidden width 16, 2 hidden layers, 1 output channel(s)
#define VPG_DEFINE_VARIANT
#include "variant.h"
namespace vpg {
VPG_DEFINE(16, 2, 1)
}  // namespace vpg

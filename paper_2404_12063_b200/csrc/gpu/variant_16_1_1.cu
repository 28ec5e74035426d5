// step kernels instantiated for hidden width 16, 1 hidden layers, 1 output channel(s)
#define VPG_DEFINE_VARIANT
#include "variant.h"
namespace vpg {
VPG_DEFINE(16, 1, 1)
}  // namespace vpg

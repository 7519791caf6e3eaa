// iterate_reg_y4.cu -- instantiations of the persistent kernel: resident slab in a register tile,
// K++, y placement 4 (see iterate_kernel.cuh).
#include "iterate_kernel.cuh"

namespace kpp {
using KernelFn = void (*)(const IterParams);
KernelFn iterate_pick_reg_y4(int rpw, int cpl) {
#define K(R, C) \
  if (rpw == R && cpl == C) return itk::iterate_kernel<1, R, C, 4, 0>;
  K(2, 1) K(4, 1) K(8, 1) K(16, 1) K(2, 2) K(4, 2) K(8, 2) K(16, 2)
#undef K
  return nullptr;
}
}  // namespace kpp

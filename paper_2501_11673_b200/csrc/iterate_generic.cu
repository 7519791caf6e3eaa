// iterate_generic.cu -- instantiations of the persistent kernel without a register tile: resident
// slab read from shared memory (any s, CD++) and streaming from HBM (c4/c5-sized blocks).
#include "iterate_kernel.cuh"

namespace kpp {
using KernelFn = void (*)(const IterParams);
KernelFn iterate_pick_generic(int resident, int yg, int cd) {
#define K(RS, Y, CD) \
  if (resident == RS && yg == Y && cd == CD) return itk::iterate_kernel<RS, 0, 0, Y, CD>;
  K(1, 0, 0) K(1, 1, 0) K(1, 4, 0) K(1, 0, 1) K(1, 1, 1) K(1, 4, 1)
  K(0, 0, 0) K(0, 1, 0) K(0, 0, 1) K(0, 1, 1)
#undef K
  return nullptr;
}
}  // namespace kpp

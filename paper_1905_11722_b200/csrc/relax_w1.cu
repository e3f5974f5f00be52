// relax_w1.cu — relaxation kernels and drivers for 1-word bitsets.
#include "relax_decl.h"
#include "relax_impl.cuh"

namespace remat {
REMAT_INSTANTIATE_RELAX(1)
}  // namespace remat

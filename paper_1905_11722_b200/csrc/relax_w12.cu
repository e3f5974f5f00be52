// relax_w12.cu — relaxation kernels and drivers for 12-word bitsets.
#include "relax_decl.h"
#include "relax_impl.cuh"

namespace remat {
REMAT_INSTANTIATE_RELAX(12)
}  // namespace remat

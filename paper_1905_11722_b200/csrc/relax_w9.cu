// relax_w9.cu — relaxation kernels and drivers for 9-word bitsets.
#include "relax_decl.h"
#include "relax_impl.cuh"

namespace remat {
REMAT_INSTANTIATE_RELAX(9)
}  // namespace remat

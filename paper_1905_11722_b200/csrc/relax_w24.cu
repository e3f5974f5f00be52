// relax_w24.cu — relaxation kernels and drivers for 24-word bitsets.
#include "relax_decl.h"
#include "relax_impl.cuh"

namespace remat {
REMAT_INSTANTIATE_RELAX(24)
}  // namespace remat

// relax_w32.cu — relaxation kernels and drivers for 32-word bitsets.
#include "relax_decl.h"
#include "relax_impl.cuh"

namespace remat {
REMAT_INSTANTIATE_RELAX(32)
}  // namespace remat

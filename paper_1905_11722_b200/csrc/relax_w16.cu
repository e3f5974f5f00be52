// relax_w16.cu — relaxation kernels and drivers for 16-word bitsets.
#include "relax_decl.h"
#include "relax_impl.cuh"

namespace remat {
REMAT_INSTANTIATE_RELAX(16)
}  // namespace remat

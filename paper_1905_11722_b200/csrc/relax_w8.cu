// relax_w8.cu — relaxation kernels and drivers for 8-word bitsets.
#include "relax_decl.h"
#include "relax_impl.cuh"

namespace remat {
REMAT_INSTANTIATE_RELAX(8)
}  // namespace remat

// relax_w6.cu — relaxation kernels and drivers for 6-word bitsets.
#include "relax_decl.h"
#include "relax_impl.cuh"

namespace remat {
REMAT_INSTANTIATE_RELAX(6)
}  // namespace remat

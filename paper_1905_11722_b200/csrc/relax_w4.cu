// relax_w4.cu — relaxation kernels and drivers for 4-word bitsets.
#include "relax_decl.h"
#include "relax_impl.cuh"

namespace remat {
REMAT_INSTANTIATE_RELAX(4)
}  // namespace remat

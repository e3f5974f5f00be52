// relax_w3.cu — relaxation kernels and drivers for 3-word bitsets.
#include "relax_decl.h"
#include "relax_impl.cuh"

namespace remat {
REMAT_INSTANTIATE_RELAX(3)
}  // namespace remat

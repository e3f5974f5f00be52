// relax_w2.cu — relaxation kernels and drivers for 2-word bitsets.
#include "relax_decl.h"
#include "relax_impl.cuh"

namespace remat {
REMAT_INSTANTIATE_RELAX(2)
}  // namespace remat

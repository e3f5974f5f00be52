// relax_w9.cu — relaxation kernels and drivers for 9-word bitsets.
#include "relax_decl.h"
#include "relax_impl.cuh"

namespace remat {
REMAT_INSTANTIATE_RELAX(9)
}  // namespace remat

#ifdef REMAT_RELAX_TRACE
namespace remat {
extern "C" __attribute__((visibility("default"))) int remat_debug_relax_trace(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_relax_trace, sizeof(g_relax_trace)) == cudaSuccess ? 0 : -1;
}
}  // namespace remat
#endif

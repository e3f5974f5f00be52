// Microbenchmark: cost of a cooperative-groups grid barrier on this GPU
// (blocks = SMs x {1,2,4}), and of a barrier + one dependent L2 round trip.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k_sync(int iters, unsigned long long* sink, int touch) {
  cg::grid_group g = cg::this_grid();
  unsigned long long acc = 0;
  for (int i = 0; i < iters; i++) {
    if (touch && threadIdx.x == 0) acc += atomicAdd(sink + (i & 7), 1ull);
    g.sync();
  }
  if (threadIdx.x == 0 && acc == 42) sink[9] = acc;
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* sink;
  cudaMalloc(&sink, 128);
  for (int touch = 0; touch < 2; touch++)
    for (int bps : {1, 2, 4}) {
      int iters = 2000;
      void* args[] = {&iters, &sink, &touch};
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaLaunchCooperativeKernel((void*)k_sync, sms * bps, 256, args, 0, 0);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_sync, sms * bps, 256, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("blocks=%d atomic_round_trip=%d: %.2f us per grid barrier\n", sms * bps, touch,
             1e3f * ms / iters);
    }
  return 0;
}

// Microbenchmark: per-SM throughput of the instruction classes the relaxation
// inner loop is made of (MEASURED_PEAKS.json has only HBM and
// bf16 figures).  Prints one JSON line:
//   int32 ALU ops/s (IADD3/LOP3 on independent chains),
//   shared RED.MIN.u32 per second (conflict-free lanes),
//   shared LDS.128 per second (broadcast-free, conflict-free),
// each also as warp-instructions per clock per SM at the measured clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/pipes tools/micro/pipes.cu
#include <cstdio>

__global__ void __launch_bounds__(256) k_alu(int iters, unsigned* out) {
  unsigned a0 = threadIdx.x, a1 = a0 ^ 1, a2 = a0 ^ 2, a3 = a0 ^ 3, a4 = a0 ^ 4, a5 = a0 ^ 5,
           a6 = a0 ^ 6, a7 = a0 ^ 7;
  const unsigned k = blockIdx.x | 1;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int r = 0; r < 16; r++) {  // 8 chains x 2 ops x 16 = 256 ops per iteration
      a0 = (a0 + k) ^ a1; a1 = (a1 + k) ^ a2; a2 = (a2 + k) ^ a3; a3 = (a3 + k) ^ a4;
      a4 = (a4 + k) ^ a5; a5 = (a5 + k) ^ a6; a6 = (a6 + k) ^ a7; a7 = (a7 + k) ^ a0;
    }
  }
  if ((a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7) == 0x12345678u) out[0] = 1;
}

__global__ void __launch_bounds__(256) k_red(int iters, unsigned* out) {
  __shared__ unsigned row[8 * 1024];
  for (int i = threadIdx.x; i < 8 * 1024; i += 256) row[i] = 0xffffffffu;
  __syncthreads();
  const unsigned base = (unsigned)__cvta_generic_to_shared(row) + 4u * threadIdx.x;
  unsigned key = 0x7fffffffu - threadIdx.x;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int r = 0; r < 16; r++) {
      asm volatile("red.shared.min.u32 [%0], %1;" ::"r"(base + 1024u * ((r + i) & 7)), "r"(key)
                   : "memory");
      key -= 1;
    }
  }
  __syncthreads();
  if (row[threadIdx.x] == 1u) out[0] = 1;
}

__global__ void __launch_bounds__(256) k_lds(int iters, unsigned* out) {
  __shared__ uint4 q[8 * 256];
  for (int i = threadIdx.x; i < 8 * 256; i += 256) q[i] = make_uint4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  unsigned acc = 0;
  const unsigned base = (unsigned)__cvta_generic_to_shared(q) + 16u * (threadIdx.x & 255);
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int r = 0; r < 16; r++) {
      uint4 v;
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                   : "r"(base + 4096u * ((r + i) & 7))
                   : "memory");
      acc += (v.x ^ v.w) + (v.y ^ v.z);
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <typename K>
static double time_ms(K kern, int blocks, int iters, unsigned* out) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kern<<<blocks, 256>>>(iters, out);  // warm-up
  cudaEventRecord(a);
  kern<<<blocks, 256>>>(iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  int sms = 0, clk_khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  unsigned* out;
  cudaMalloc(&out, 64);
  const int blocks = sms * 8, iters = 4096;
  const double threads = (double)blocks * 256;
  const double ms_alu = time_ms(k_alu, blocks, iters, out);
  const double ms_red = time_ms(k_red, blocks, iters, out);
  const double ms_lds = time_ms(k_lds, blocks, iters, out);
  const double alu_ops = threads * iters * 256 / (ms_alu * 1e-3);
  const double reds = threads * iters * 16 / (ms_red * 1e-3);
  const double lds = threads * iters * 16 / (ms_lds * 1e-3);
  const double per_clk = 1.0 / (sms * (clk_khz * 1e3) * 32);  // warp-instr per clock per SM
  printf("{\"sms\": %d, \"clock_mhz\": %.0f, \"int32_ops_per_s\": %.4g, \"int32_warp_ops_per_clk_sm\": %.3f, "
         "\"red_shared_per_s\": %.4g, \"red_shared_warp_per_clk_sm\": %.3f, "
         "\"lds128_per_s\": %.4g, \"lds128_warp_per_clk_sm\": %.3f}\n",
         sms, clk_khz / 1e3, alu_ops, alu_ops * per_clk, reds, reds * per_clk, lds, lds * per_clk);
  return 0;
}

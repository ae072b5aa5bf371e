// Microbenchmark: Philox4x32-10 calls per second on the whole GPU (the keep-flag generator
// of the dropout sites, common.cuh) at several occupancies -- the FMA-pipe cost of the
// 32x32->64 multiplies that bounds in-kernel mask generation.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o philox_rate philox_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2007_00072_b200/csrc/common.cuh"
using namespace enc;

template <int ILP>
__global__ void philox_kernel(uint32_t* out, int64_t calls, PhiloxKey pk) {
  uint32_t acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * ILP;
  for (int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * ILP; g < calls; g += stride) {
#pragma unroll
    for (int j = 0; j < ILP; ++j) {
      const uint4 w = philox4x32_10((uint64_t)(g + j), pk);
      acc ^= w.x ^ w.y ^ w.z ^ w.w;
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  PhiloxKey pk{};
  for (int r = 0; r < 10; ++r) { pk.rk0[r] = 0x9E3779B9u * r + 1; pk.rk1[r] = 0xBB67AE85u * r + 7; }
  pk.a0 = 3; pk.l1 = 5; pk.b0 = 7; pk.T = 6554; pk.scale = 1.1f;
  uint32_t* out; cudaMalloc(&out, 4);
  const int64_t calls = 4194304LL * 8;   // 8x the attention mask of config L
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int threads : {128, 256, 512, 1024}) {
    for (int ilp : {1, 2, 4}) {
      auto run = [&]() {
        if (ilp == 1) philox_kernel<1><<<sms, threads>>>(out, calls, pk);
        if (ilp == 2) philox_kernel<2><<<sms, threads>>>(out, calls, pk);
        if (ilp == 4) philox_kernel<4><<<sms, threads>>>(out, calls, pk);
      };
      run(); cudaDeviceSynchronize();
      cudaEventRecord(e0); run(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double per_smsp_cycles = ms * 1e-3 * clk * 1e3 / 1.0;   // cycles elapsed
      const double warp_calls_per_smsp = (double)calls / 32 / (sms * 4);
      printf("threads/SM %4d ILP %d: %.2f us for %lld calls -> %.1f SMSP cycles per warp-call "
             "(%.2f us per 4.19 M calls)\n", threads, ilp, ms * 1e3, (long long)calls,
             per_smsp_cycles / warp_calls_per_smsp, ms * 1e3 / 8);
    }
  }
  return 0;
}

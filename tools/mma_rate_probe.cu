// Issue-to-completion time of a chain of cta_group::1 bf16 tcgen05.mma instructions, one CTA
// per SM, by operand form: A from TMEM (TS) or shared memory (SS), B K-major or MN-major
// (SWIZZLE_128B), N = 64 or 256.  Debug tool for the fused score + A.V kernel's C = A V step.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17
//        -I paper_2007_00072_b200/csrc -o tools/mma_rate_probe tools/mma_rate_probe.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdio.h>

#include "tc_gemm.cuh"

using namespace enc;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc));
}

// mode: 0 TS N=64 B MN-major (the fused kernel's A.V), 1 SS N=64 B MN-major,
//       2 SS N=64 B K-major, 3 TS N=64 B K-major, 4 SS N=256 B K-major (the score MMA),
//       5 TS N=256 B K-major, 6/7/8 mode 0 spread over 2/4/8 accumulators (8: N=32 halves)
// unrolled chain with the descriptors formed outside the timed loop: N, accumulators, TS
template <int N, int NACC, bool TS>
__device__ __forceinline__ void chain32(uint32_t tmem, uint32_t a0, uint32_t b0) {
  const uint64_t bd = tc::smem_desc(b0, 8192, 1024);
  const uint64_t ad = tc::smem_desc(a0, 16, 1024);
  constexpr uint32_t idesc = tc::instr_desc_bf16_f32(128, N, false, true);
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const uint32_t d = tmem + 256 + N * (k % NACC);
    if (TS)
      mma_ts(d, tmem + 8 * k, bd + (uint64_t)((k * 2048) >> 4), idesc, k >= NACC);
    else
      tc::mma_bf16(d, ad + (uint64_t)(((k & 3) * 32 + (k >> 2 & 3) * 16384) >> 4),
                   bd + (uint64_t)((k * 2048) >> 4), idesc, k >= NACC);
  }
}

__global__ void probe(unsigned long long* out, int mode, int n_mma) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 160 * 1024);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc(slot, 512);
  fence_proxy_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *slot;
  const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 64 * 1024);
  unsigned long long best = ~0ull;
  for (int rep = 0; rep < 8; ++rep) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const long long t0 = clock64();
      if (mode >= 9) {
        switch (mode) {
          case 9: chain32<64, 1, true>(tmem, a0, b0); break;
          case 10: chain32<64, 2, true>(tmem, a0, b0); break;
          case 11: chain32<64, 4, true>(tmem, a0, b0); break;
          case 12: chain32<64, 1, false>(tmem, a0, b0); break;
          case 13: chain32<128, 1, true>(tmem, a0, b0); break;
          default: chain32<256, 1, true>(tmem, a0, b0); break;
        }
      }
      for (int k = 0; k < (mode >= 9 ? 0 : n_mma); ++k) {
        const uint32_t acc = k != 0;
        switch (mode) {
          case 0:
            mma_ts(tmem + 256, tmem + 8 * (k & 31), tc::smem_desc(b0 + (k & 31) * 2048, 8192, 1024),
                   tc::instr_desc_bf16_f32(128, 64, false, true), acc);
            break;
          case 1:
            tc::mma_bf16(tmem + 256, tc::smem_desc(a0 + (k & 3) * 32 + (k >> 2 & 3) * 16384, 16, 1024),
                         tc::smem_desc(b0 + (k & 31) * 2048, 8192, 1024),
                         tc::instr_desc_bf16_f32(128, 64, false, true), acc);
            break;
          case 2:
            tc::mma_bf16(tmem + 256, tc::smem_desc(a0 + (k & 3) * 32 + (k >> 2 & 3) * 16384, 16, 1024),
                         tc::smem_desc(b0 + (k & 3) * 32, 16, 1024),
                         tc::instr_desc_bf16_f32(128, 64, false, false), acc);
            break;
          case 3:
            mma_ts(tmem + 256, tmem + 8 * (k & 31), tc::smem_desc(b0 + (k & 3) * 32, 16, 1024),
                   tc::instr_desc_bf16_f32(128, 64, false, false), acc);
            break;
          case 4:
            tc::mma_bf16(tmem + 256, tc::smem_desc(a0 + (k & 3) * 32, 16, 1024),
                         tc::smem_desc(b0 + (k & 3) * 32, 16, 1024),
                         tc::instr_desc_bf16_f32(128, 256, false, false), acc);
            break;
          case 5:
            mma_ts(tmem + 256, tmem + 8 * (k & 31), tc::smem_desc(b0 + (k & 3) * 32, 16, 1024),
                   tc::instr_desc_bf16_f32(128, 256, false, false), acc);
            break;
          default: {   // 6 / 7 / 8: A.V of mode 0 over 2 / 4 / 8 accumulators (k-step k -> k % nacc)
            const int nacc = mode == 6 ? 2 : mode == 7 ? 4 : 8;
            const int acc_i = k % nacc;
            mma_ts(tmem + 256 + (nacc == 8 ? 32 : 64) * acc_i, tmem + 8 * (k & 31),
                   tc::smem_desc(b0 + (k & 31) * 2048, 8192, 1024),
                   tc::instr_desc_bf16_f32(128, nacc == 8 ? 32 : 64, false, true), k >= nacc);
            break;
          }
        }
      }
      tc::mma_commit(bar);
      mbar_wait(bar, rep & 1);
      const long long t1 = clock64();
      if ((unsigned long long)(t1 - t0) < best) best = t1 - t0;
    }
  }
  if (threadIdx.x == 0) out[blockIdx.x] = best;
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * sizeof(unsigned long long));
  const size_t smem = 160 * 1024 + 2048;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const char* names[] = {"TS  N=64  B MN-major", "SS  N=64  B MN-major", "SS  N=64  B K-major",
                         "TS  N=64  B K-major", "SS  N=256 B K-major", "TS  N=256 B K-major", "TS  N=64 MN 2 acc    ", "TS  N=64 MN 4 acc    ",
                         "TS  N=32 MN 8 acc    ", "unrolled TS N=64 1acc", "unrolled TS N=64 2acc",
                         "unrolled TS N=64 4acc", "unrolled SS N=64 1acc", "unrolled TS N=128   ",
                         "unrolled TS N=256   "};
  for (int grid : {148})
    for (int mode = 0; mode < 15; ++mode)
      for (int n : {8, 32}) {
        if (mode >= 9 && n != 32) continue;
        probe<<<grid, 128, smem>>>(d, mode, n);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[148];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        unsigned long long mx = 0;
        for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("grid %3d  %s  %2d MMAs: %6llu cycles (%5.1f per MMA)  %s\n", grid, names[mode], n,
               mx, (double)mx / n, cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
      }
  return 0;
}

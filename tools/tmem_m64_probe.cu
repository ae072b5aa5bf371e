// Where does a cta_group::1 tcgen05.mma with M = 64 put its accumulator rows in TMEM, and
// may its destination start at TMEM lane 64?  A[r][0] = r+1 (first MMA, D at lane 0) and
// 101+r (second MMA, D at lane 64), B[n][0] = 1, so D[r][n] = A[r][0].  Every thread
// then reads TMEM columns 0 and 1 of its lane and writes them out.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17
//        -I paper_2007_00072_b200/csrc -o tools/tmem_m64_probe tools/tmem_m64_probe.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdio.h>

#include "tc_gemm.cuh"

using namespace enc;

__global__ void probe(float* out, int second_at_lane64) {
  __shared__ __align__(1024) unsigned char smem[2 * 8192 + 16384 + 64];
  unsigned char* A0 = smem;            // 64 rows x 128 B
  unsigned char* A1 = smem + 8192;
  unsigned char* Bm = smem + 16384;    // 128 rows x 128 B
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384 + 16384);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < (2 * 8192 + 16384) / 2; i += blockDim.x)
    reinterpret_cast<__nv_bfloat16*>(smem)[i] = __float2bfloat16(0.f);
  __syncthreads();
  if (threadIdx.x < 64) {
    const int r = threadIdx.x;
    const int off = r * 128 + ((0 ^ (r & 7)) << 4);
    *reinterpret_cast<__nv_bfloat16*>(A0 + off) = __float2bfloat16((float)(r + 1));
    *reinterpret_cast<__nv_bfloat16*>(A1 + off) = __float2bfloat16((float)(101 + r));
  }
  for (int n = threadIdx.x; n < 128; n += blockDim.x)
    *reinterpret_cast<__nv_bfloat16*>(Bm + n * 128 + ((0 ^ (n & 7)) << 4)) = __float2bfloat16(1.f);
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
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = tc::instr_desc_bf16_f32(64, 128, false, false);
    for (int k = 0; k < 4; ++k)
      tc::mma_bf16(tmem, tc::smem_desc(smem_u32(A0) + k * 32, 16, 1024),
                   tc::smem_desc(smem_u32(Bm) + k * 32, 16, 1024), idesc, k != 0);
    // mode 0: second D at column 256; 1: at lane 64; 2: at lane 16 (same columns)
    const uint32_t d2 = second_at_lane64 == 1   ? tmem + (64u << 16)
                        : second_at_lane64 == 2 ? tmem + (16u << 16)
                                                : tmem + 256;
    for (int k = 0; k < 4; ++k)
      tc::mma_bf16(d2, tc::smem_desc(smem_u32(A1) + k * 32, 16, 1024),
                   tc::smem_desc(smem_u32(Bm) + k * 32, 16, 1024), idesc, k != 0);
    tc::mma_commit(bar);
  }
  __syncwarp();
  mbar_wait(bar, 0);
  tc::fence_after_sync();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float v[32];
  tc::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16), v);
  out[threadIdx.x * 4 + 0] = v[0];
  out[threadIdx.x * 4 + 1] = v[1];
  tc::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + 256, v);
  out[threadIdx.x * 4 + 2] = v[0];
  out[threadIdx.x * 4 + 3] = v[1];
  (void)lane;
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc(tmem, 512);
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 4 * sizeof(float));
  for (int mode = 0; mode < 3; ++mode) {
    cudaMemset(d, 0, 128 * 4 * sizeof(float));
    probe<<<1, 128>>>(d, mode);
    cudaError_t e = cudaDeviceSynchronize();
    float h[512];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("mode %d (second MMA at %s): %s\n", mode,
           mode == 1 ? "lane 64" : mode == 2 ? "lane 16" : "column 256",
           cudaGetErrorString(e));
    for (int t = 0; t < 128; t += 4)
      printf("  lane %3d: col0 %6.1f col1 %6.1f | col256 %6.1f col257 %6.1f   lane %3d: %6.1f %6.1f | %6.1f %6.1f\n",
             t, h[t * 4], h[t * 4 + 1], h[t * 4 + 2], h[t * 4 + 3], t + 1, h[(t + 1) * 4],
             h[(t + 1) * 4 + 1], h[(t + 1) * 4 + 2], h[(t + 1) * 4 + 3]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}

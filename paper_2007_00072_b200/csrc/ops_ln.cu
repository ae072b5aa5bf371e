// BDRLN: bias + dropout + residual + LayerNorm (paper `drln`/`bdrln`) and
// its backward (paper `bsb` + `blnrd` + `ebsb` + `baob`), plus
// the deterministic column-sum finalize shared by all bias/gamma/beta reductions.
//
// One warp per row of I elements held in registers; mean and variance are warp-shuffle
// all-reductions (two passes over registers, no re-read).  The backward accumulates the
// three column sums (dgamma, dbeta, dbias) in registers across the rows a warp visits,
// reduces them across the CTA's warps in a fixed order through shared memory and writes
// one partial row per CTA; launch_colsum_finalize sums the partial rows in a fixed
// order.  No float atomics: results are bitwise reproducible run to run.
#include <math.h>

#include "kernels.h"

namespace enc {

// ------------------------------------------------------------------ BDRLN forward
template <typename T, int CPL>
__global__ void __launch_bounds__(256) bdrln_fwd_kernel(
    const T* __restrict__ Y, const float* __restrict__ bias, const T* __restrict__ R,
    const float* __restrict__ gamma, const float* __restrict__ beta, T* __restrict__ out,
    T* __restrict__ xhat, float* __restrict__ rstd_out, int rows, int I, float eps, int64_t g0,
    PhiloxKey pk) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int nc = I >> 3;
  const int64_t base = (int64_t)row * I;
  float z[CPL][8];
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < CPL; ++i) {
    const int ch = lane + 32 * i;
    if (ch < nc) {
      float y[8], b[8];
      Chunk<T>::load_cs(Y + base + ch * 8, y);
      Chunk<T>::load_cs(R + base + ch * 8, z[i]);
      load_f32x8(bias + ch * 8, b);
      const uint32_t kb = keep_bits8((uint64_t)(g0 + (int64_t)row * nc + ch), pk);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        z[i][j] += ((kb >> j) & 1u) ? (y[j] + b[j]) * pk.scale : 0.f;
        sum += z[i][j];
      }
    }
  }
  const float inv_n = 1.f / (float)I;
  const float mean = warp_sum(sum) * inv_n;
  float sq = 0.f;
#pragma unroll
  for (int i = 0; i < CPL; ++i) {
    if (lane + 32 * i < nc) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float d = z[i][j] - mean;
        sq = fmaf(d, d, sq);
      }
    }
  }
  const float var = warp_sum(sq) * inv_n;
  const float rstd = rsqrtf(var + eps);
#pragma unroll
  for (int i = 0; i < CPL; ++i) {
    const int ch = lane + 32 * i;
    if (ch < nc) {
      float g[8], be[8], xh[8], o[8];
      load_f32x8(gamma + ch * 8, g);
      load_f32x8(beta + ch * 8, be);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        xh[j] = (z[i][j] - mean) * rstd;
        o[j] = fmaf(g[j], xh[j], be[j]);
      }
      Chunk<T>::store(out + base + ch * 8, o);
      Chunk<T>::store(xhat + base + ch * 8, xh);
    }
  }
  if (lane == 0) rstd_out[row] = rstd;
}

cudaError_t launch_bdrln_fwd(int dtype, int B, int J, int I, const void* Y, const float* bias,
                             const void* R, const float* gamma, const float* beta, float eps,
                             const PhiloxKey& pk, int64_t batch_offset, void* out, void* xhat,
                             float* rstd, cudaStream_t st) {
  const int rows = B * J;
  if (rows == 0) return cudaSuccess;
  const int nc = I / 8;
  const int64_t g0 = batch_offset * (int64_t)J * nc;
  const int grid = (rows + 7) / 8;
  ENC_CPL_DISPATCH(nc, {
    if (dtype == 0)
      bdrln_fwd_kernel<__nv_bfloat16, CPL><<<grid, 256, 0, st>>>(
          (const __nv_bfloat16*)Y, bias, (const __nv_bfloat16*)R, gamma, beta,
          (__nv_bfloat16*)out, (__nv_bfloat16*)xhat, rstd, rows, I, eps, g0, pk);
    else
      bdrln_fwd_kernel<float, CPL><<<grid, 256, 0, st>>>(
          (const float*)Y, bias, (const float*)R, gamma, beta, (float*)out, (float*)xhat, rstd,
          rows, I, eps, g0, pk);
  });
  return cudaGetLastError();
}

// ------------------------------------------------------------------ BDRLN backward
constexpr int kLnBwdWarps = 8;

template <typename T, int CPL>
__global__ void __launch_bounds__(256) bdrln_bwd_kernel(
    const T* __restrict__ dOut, const T* __restrict__ xhat, const float* __restrict__ rstd,
    const float* __restrict__ gamma, T* __restrict__ dz, T* __restrict__ dYpre,
    float* __restrict__ partials, int rows, int I, int64_t g0, PhiloxKey pk) {
  extern __shared__ float red[];  // [3][I]
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nc = I >> 3;
  const float inv_n = 1.f / (float)I;
  float acc_g[CPL][8], acc_b[CPL][8], acc_d[CPL][8];
#pragma unroll
  for (int i = 0; i < CPL; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc_g[i][j] = acc_b[i][j] = acc_d[i][j] = 0.f;

  const int stride = gridDim.x * kLnBwdWarps;
  for (int row = blockIdx.x * kLnBwdWarps + warp; row < rows; row += stride) {
    const int64_t base = (int64_t)row * I;
    float go[CPL][8], xh[CPL][8];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
      const int ch = lane + 32 * i;
      if (ch < nc) {
        float gm[8];
        Chunk<T>::load_cs(dOut + base + ch * 8, go[i]);
        Chunk<T>::load_cs(xhat + base + ch * 8, xh[i]);
        load_f32x8(gamma + ch * 8, gm);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          acc_g[i][j] = fmaf(go[i][j], xh[i][j], acc_g[i][j]);
          acc_b[i][j] += go[i][j];
          go[i][j] *= gm[j];  // g = dOut * gamma
          s1 += go[i][j];
          s2 = fmaf(go[i][j], xh[i][j], s2);
        }
      }
    }
    const float mg = warp_sum(s1) * inv_n;
    const float mgx = warp_sum(s2) * inv_n;
    const float rs = __ldg(rstd + row);
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
      const int ch = lane + 32 * i;
      if (ch < nc) {
        float d[8], y[8];
        const uint32_t kb = keep_bits8((uint64_t)(g0 + (int64_t)row * nc + ch), pk);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          d[j] = rs * (go[i][j] - mg - xh[i][j] * mgx);
          y[j] = ((kb >> j) & 1u) ? d[j] * pk.scale : 0.f;
          acc_d[i][j] += y[j];
        }
        Chunk<T>::store(dz + base + ch * 8, d);
        Chunk<T>::store(dYpre + base + ch * 8, y);
      }
    }
  }
  // fixed-order CTA reduction: warp 0 writes, warps 1..7 add in turn
  for (int w = 0; w < kLnBwdWarps; ++w) {
    if (warp == w) {
#pragma unroll
      for (int i = 0; i < CPL; ++i) {
        const int ch = lane + 32 * i;
        if (ch < nc) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int c = ch * 8 + j;
            if (w == 0) {
              red[c] = acc_g[i][j];
              red[I + c] = acc_b[i][j];
              red[2 * I + c] = acc_d[i][j];
            } else {
              red[c] += acc_g[i][j];
              red[I + c] += acc_b[i][j];
              red[2 * I + c] += acc_d[i][j];
            }
          }
        }
      }
    }
    __syncthreads();
  }
  float* out = partials + (int64_t)blockIdx.x * 3 * I;
  for (int c = threadIdx.x; c < 3 * I; c += blockDim.x) out[c] = red[c];
}

cudaError_t launch_bdrln_bwd(int dtype, int B, int J, int I, const void* dOut, const void* xhat,
                             const float* rstd, const float* gamma, const PhiloxKey& pk,
                             int64_t batch_offset, void* dz, void* dYpre, float* dgamma,
                             float* dbeta, float* dbias, const ReduceWs& ws, cudaStream_t st) {
  const int rows = B * J;
  if (rows == 0) {
    cudaMemsetAsync(dgamma, 0, sizeof(float) * I, st);
    cudaMemsetAsync(dbeta, 0, sizeof(float) * I, st);
    return cudaMemsetAsync(dbias, 0, sizeof(float) * I, st);
  }
  const int nc = I / 8;
  const int64_t g0 = batch_offset * (int64_t)J * nc;
  // ~2 rows per warp: enough CTAs to cover every SM, few partial rows
  int G = (rows + 2 * kLnBwdWarps - 1) / (2 * kLnBwdWarps);
  if (G > 2 * ws.num_sms) G = 2 * ws.num_sms;
  const size_t cap = ws.cap_floats / (size_t)(3 * I);
  if ((size_t)G > cap) G = (int)cap;
  if (G < 1) G = 1;
  const size_t smem = sizeof(float) * 3 * I;
  ENC_CPL_DISPATCH(nc, {
    if (dtype == 0) {
      auto kern = bdrln_bwd_kernel<__nv_bfloat16, CPL>;
      if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kern<<<G, 256, smem, st>>>((const __nv_bfloat16*)dOut, (const __nv_bfloat16*)xhat, rstd,
                                 gamma, (__nv_bfloat16*)dz, (__nv_bfloat16*)dYpre, ws.partials,
                                 rows, I, g0, pk);
    } else {
      auto kern = bdrln_bwd_kernel<float, CPL>;
      if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kern<<<G, 256, smem, st>>>((const float*)dOut, (const float*)xhat, rstd, gamma,
                                 (float*)dz, (float*)dYpre, ws.partials, rows, I, g0, pk);
    }
  });
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_colsum_finalize(ws.partials, G, 3 * I, I, dgamma, dbeta, dbias, st);
}

// ------------------------------------------------------------------ column-sum finalize
// Block (32 columns) x (16 row-slices).  Thread (x, y) sums partial rows y, y+16, ... of
// column c in ascending order; the 16 slice sums are then added in ascending y order.
constexpr int kFinY = 16;

__global__ void __launch_bounds__(32 * kFinY) colsum_finalize_kernel(
    const float* __restrict__ partials, int R, int ncols, int nper, float* out0, float* out1,
    float* out2) {
  __shared__ float sm[kFinY][33];
  const int c = blockIdx.x * 32 + threadIdx.x;
  float s = 0.f;
  if (c < ncols) {
#pragma unroll 8
    for (int r = threadIdx.y; r < R; r += kFinY) s += partials[(int64_t)r * ncols + c];
  }
  sm[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.y == 0 && c < ncols) {
    float t = sm[0][threadIdx.x];
#pragma unroll
    for (int y = 1; y < kFinY; ++y) t += sm[y][threadIdx.x];
    const int q = c / nper;
    const int j = c - q * nper;
    float* o = q == 0 ? out0 : (q == 1 ? out1 : out2);
    o[j] = t;
  }
}

cudaError_t launch_colsum_finalize(const float* partials, int R, int ncols, int nper,
                                   float* out0, float* out1, float* out2, cudaStream_t st) {
  dim3 block(32, kFinY);
  colsum_finalize_kernel<<<(ncols + 31) / 32, block, 0, st>>>(partials, R, ncols, nper, out0,
                                                              out1, out2);
  return cudaGetLastError();
}

}  // namespace enc

// BAD: bias + activation + dropout (paper `brd`) and its backward (paper
// `bdrb`), plus BEI (paper `bei`).
//
// BAD forward is element-wise: one thread per 8-element chunk (a 16-byte bf16 vector),
// grid-stride.  BAD backward is element-wise plus a column reduction (db1): it is laid
// out column-parallel -- a thread owns one chunk column and walks a block of rows, so
// the bias-gradient partial stays in 8 registers and each warp still reads/writes 512
// contiguous bytes per row.
#include <math.h>

#include "kernels.h"

namespace enc {

enum { kActGeluErf = 0, kActGeluTanh = 1, kActRelu = 2 };

template <int ACT>
__device__ __forceinline__ float act_f(float h) {
  if (ACT == kActGeluErf) return 0.5f * h * (1.f + erff(h * 0.70710678118654752f));
  if (ACT == kActGeluTanh) {
    const float u = 0.7978845608028654f * (h + 0.044715f * h * h * h);
    return 0.5f * h * (1.f + tanhf(u));
  }
  return h > 0.f ? h : 0.f;
}

template <int ACT>
__device__ __forceinline__ float act_df(float h) {
  if (ACT == kActGeluErf)
    return 0.5f * (1.f + erff(h * 0.70710678118654752f)) +
           h * 0.3989422804014327f * __expf(-0.5f * h * h);
  if (ACT == kActGeluTanh) {
    const float c = 0.7978845608028654f;
    const float t = tanhf(c * (h + 0.044715f * h * h * h));
    return 0.5f * (1.f + t) + 0.5f * h * (1.f - t * t) * c * (1.f + 3.f * 0.044715f * h * h);
  }
  return h > 0.f ? 1.f : 0.f;
}

// ------------------------------------------------------------------ BAD forward
template <typename T, int ACT>
__global__ void __launch_bounds__(256) bad_fwd_kernel(const T* __restrict__ Y1,
                                                      const float* __restrict__ b1,
                                                      T* __restrict__ h_out,
                                                      T* __restrict__ A1, int64_t nchunks,
                                                      int ncU, int64_t g0, PhiloxKey pk) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nchunks;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int col = (int)(c % ncU) << 3;
    float y[8], b[8], a[8];
    Chunk<T>::load_cs(Y1 + c * 8, y);
    load_f32x8(b1 + col, b);
    const uint32_t kb = keep_bits8((uint64_t)(g0 + c), pk);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      y[j] += b[j];
      a[j] = ((kb >> j) & 1u) ? act_f<ACT>(y[j]) * pk.scale : 0.f;
    }
    Chunk<T>::store(h_out + c * 8, y);
    Chunk<T>::store(A1 + c * 8, a);
  }
}

#define ENC_ACT_DISPATCH(act, ...)                                      \
  do {                                                                   \
    if ((act) == kActGeluErf) { constexpr int ACT = kActGeluErf; __VA_ARGS__; }   \
    else if ((act) == kActGeluTanh) { constexpr int ACT = kActGeluTanh; __VA_ARGS__; } \
    else { constexpr int ACT = kActRelu; __VA_ARGS__; }                         \
  } while (0)

cudaError_t launch_bad_fwd(int dtype, int B, int J, int U, const void* Y1, const float* b1,
                           int act, const PhiloxKey& pk, int64_t batch_offset, void* h,
                           void* A1, cudaStream_t st) {
  const int64_t n = (int64_t)B * J * (U / 8);
  if (n == 0) return cudaSuccess;
  const int ncU = U / 8;
  const int64_t g0 = batch_offset * (int64_t)J * ncU;
  int64_t grid = (n + 255) / 256;
  if (grid > 148 * 16) grid = 148 * 16;
  ENC_ACT_DISPATCH(act, {
    if (dtype == 0)
      bad_fwd_kernel<__nv_bfloat16, ACT><<<(int)grid, 256, 0, st>>>(
          (const __nv_bfloat16*)Y1, b1, (__nv_bfloat16*)h, (__nv_bfloat16*)A1, n, ncU, g0, pk);
    else
      bad_fwd_kernel<float, ACT><<<(int)grid, 256, 0, st>>>((const float*)Y1, b1, (float*)h,
                                                            (float*)A1, n, ncU, g0, pk);
  });
  return cudaGetLastError();
}

// ------------------------------------------------------------------ BAD backward
template <typename T, int ACT>
__global__ void __launch_bounds__(128) bad_bwd_kernel(const T* __restrict__ dA1,
                                                      const T* __restrict__ h,
                                                      T* __restrict__ dh,
                                                      float* __restrict__ partials, int rows,
                                                      int rpb, int U, int64_t g0, PhiloxKey pk) {
  const int ncU = U >> 3;
  const int ch = blockIdx.x * blockDim.x + threadIdx.x;
  if (ch >= ncU) return;
  const int col = ch << 3;
  float acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = 0.f;
  const int r0 = blockIdx.y * rpb;
  const int r1 = min(rows, r0 + rpb);
#pragma unroll 2
  for (int r = r0; r < r1; ++r) {
    const int64_t off = (int64_t)r * U + col;
    float d[8], x[8];
    Chunk<T>::load_cs(dA1 + off, d);
    Chunk<T>::load_cs(h + off, x);
    const uint32_t kb = keep_bits8((uint64_t)(g0 + (int64_t)r * ncU + ch), pk);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      d[j] = ((kb >> j) & 1u) ? d[j] * pk.scale * act_df<ACT>(x[j]) : 0.f;
      acc[j] += d[j];
    }
    Chunk<T>::store(dh + off, d);
  }
  float* out = partials + (int64_t)blockIdx.y * U + col;
  reinterpret_cast<float4*>(out)[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
  reinterpret_cast<float4*>(out)[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
}

cudaError_t launch_bad_bwd(int dtype, int B, int J, int U, const void* dA1, const void* h,
                           int act, const PhiloxKey& pk, int64_t batch_offset, void* dh,
                           float* db1, const ReduceWs& ws, cudaStream_t st) {
  const int rows = B * J;
  if (rows == 0) return cudaMemsetAsync(db1, 0, sizeof(float) * U, st);
  const int ncU = U / 8;
  const int64_t g0 = batch_offset * (int64_t)J * ncU;
  const int gx = (ncU + 127) / 128;
  int R = (4 * ws.num_sms + gx - 1) / gx;
  const size_t cap = ws.cap_floats / (size_t)U;
  if ((size_t)R > cap) R = (int)cap;
  if (R > rows) R = rows;
  if (R < 1) R = 1;
  const int rpb = (rows + R - 1) / R;
  R = (rows + rpb - 1) / rpb;
  dim3 grid(gx, R);
  ENC_ACT_DISPATCH(act, {
    if (dtype == 0)
      bad_bwd_kernel<__nv_bfloat16, ACT><<<grid, 128, 0, st>>>(
          (const __nv_bfloat16*)dA1, (const __nv_bfloat16*)h, (__nv_bfloat16*)dh, ws.partials,
          rows, rpb, U, g0, pk);
    else
      bad_bwd_kernel<float, ACT><<<grid, 128, 0, st>>>((const float*)dA1, (const float*)h,
                                                       (float*)dh, ws.partials, rows, rpb, U,
                                                       g0, pk);
  });
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_colsum_finalize(ws.partials, R, U, U, db1, nullptr, nullptr, st);
}

// ------------------------------------------------------------------ BEI
template <typename T>
__global__ void __launch_bounds__(256) bei_kernel(const T* a, const T* __restrict__ b, T* out,
                                                  int64_t nchunks) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nchunks;
       c += (int64_t)gridDim.x * blockDim.x) {
    float x[8], y[8];
    Chunk<T>::load_cs(a + c * 8, x);
    Chunk<T>::load_cs(b + c * 8, y);
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] += y[j];
    Chunk<T>::store(out + c * 8, x);
  }
}

cudaError_t launch_bei(int dtype, int64_t n, const void* a, const void* b, void* out,
                       cudaStream_t st) {
  const int64_t nc = n / 8;
  if (nc == 0) return cudaSuccess;
  int64_t grid = (nc + 255) / 256;
  if (grid > 148 * 16) grid = 148 * 16;
  if (dtype == 0)
    bei_kernel<__nv_bfloat16><<<(int)grid, 256, 0, st>>>(
        (const __nv_bfloat16*)a, (const __nv_bfloat16*)b, (__nv_bfloat16*)out, nc);
  else
    bei_kernel<float><<<(int)grid, 256, 0, st>>>((const float*)a, (const float*)b, (float*)out,
                                                 nc);
  return cudaGetLastError();
}

}  // namespace enc

// BAD: bias + activation + dropout (paper `brd`) and its backward (paper
// `bdrb`), plus BEI (paper `bei`).
//
// BAD forward is element-wise: one thread per 8-element chunk (a 16-byte bf16 vector),
// grid-stride.  BAD backward is element-wise plus a column reduction (db1): it is laid
// out column-parallel -- a thread owns one chunk column and walks a block of rows, so
// the bias-gradient partial stays in 8 registers and each warp still reads/writes 512
// contiguous bytes per row.
#include <math.h>

#include "act.cuh"
#include "kernels.h"

namespace enc {

// ------------------------------------------------------------------ BAD forward
template <typename T, int ACT>
__global__ void __launch_bounds__(256) bad_fwd_kernel(const T* __restrict__ Y1,
                                                      const float* __restrict__ b1,
                                                      T* __restrict__ h_out,
                                                      T* __restrict__ A1, int64_t nchunks,
                                                      int ncU, int64_t g0, PhiloxKey pk) {
  constexpr int kU = 2;  // chunks in flight per thread
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  PhiloxKey pkh = pk;
  pkh.scale *= 0.5f;
  for (int64_t c0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c0 < nchunks;
       c0 += kU * stride) {
    typename Chunk<T>::Raw raw[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (c0 + u * stride < nchunks) raw[u] = Chunk<T>::ld(Y1 + (c0 + u * stride) * 8);
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t c = c0 + u * stride;
      if (c < nchunks) {
        const int col = ((int)c % ncU) << 3;  // chunk counts < 2^31 (host-checked)
        float y[8], b[8], a[8];
        Chunk<T>::unpack(raw[u], y);
        load_f32x8(b1 + col, b);
        float m[8];   // keep ? scale / 2 : 0 (act_f2 returns 2 GELU)
        keep_mul8((uint64_t)(g0 + c), pkh, m);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          y[j] += b[j];
          a[j] = act_f2<ACT>(y[j]) * m[j];
        }
        if (h_out != nullptr) Chunk<T>::store(h_out + c * 8, y);
        Chunk<T>::store(A1 + c * 8, a);
      }
    }
  }
}


cudaError_t launch_bad_fwd(int dtype, int B, int J, int U, const void* Y1, const float* b1,
                           int act, const PhiloxKey& pk, int64_t batch_offset, void* h,
                           void* A1, cudaStream_t st) {
  const int64_t n = (int64_t)B * J * (U / 8);
  if (n == 0) return cudaSuccess;
  const int ncU = U / 8;
  const int64_t g0 = batch_offset * (int64_t)J * ncU;
  // grid-stride over the chunks with exactly the resident number of blocks (one wave: at
  // 40 registers six 256-thread blocks fit per SM, so a fixed 8-per-SM grid left a 1/3 tail)
  auto resident = [](auto kern) -> int64_t {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 256, 0);
    return (int64_t)(per < 1 ? 1 : per) * sms;
  };
  int64_t grid = (n + 511) / 512;
  ENC_ACT_DISPATCH(act, {
    if (dtype == 0) {
      auto kern = bad_fwd_kernel<__nv_bfloat16, ACT>;
      const int64_t cap = resident(kern);
      kern<<<(int)(grid < cap ? grid : cap), 256, 0, st>>>(
          (const __nv_bfloat16*)Y1, b1, (__nv_bfloat16*)h, (__nv_bfloat16*)A1, n, ncU, g0, pk);
    } else {
      auto kern = bad_fwd_kernel<float, ACT>;
      const int64_t cap = resident(kern);
      kern<<<(int)(grid < cap ? grid : cap), 256, 0, st>>>((const float*)Y1, b1, (float*)h,
                                                           (float*)A1, n, ncU, g0, pk);
    }
  });
  return cudaGetLastError();
}

// ------------------------------------------------------------------ BAD backward
// h: the activation input, or (b1 != null) the pre-bias contraction output Y1, h = Y1 + b1
template <typename T, int ACT>
__global__ void __launch_bounds__(128, sizeof(T) == 2 ? 8 : 4) bad_bwd_kernel(const T* __restrict__ dA1,
                                                      const T* __restrict__ h,
                                                      const float* __restrict__ b1,
                                                      T* __restrict__ dh,
                                                      float* __restrict__ partials, int rows,
                                                      int rpb, int U, int64_t g0, PhiloxKey pk) {
  const int ncU = U >> 3;
  const int ch = blockIdx.x * blockDim.x + threadIdx.x;
  if (ch >= ncU) return;
  const int col = ch << 3;
  float acc[8], bb[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = 0.f;
  if (b1 != nullptr)
    load_f32x8(b1 + col, bb);
  else
#pragma unroll
    for (int j = 0; j < 8; ++j) bb[j] = 0.f;
  const int r0 = blockIdx.y * rpb;
  const int r1 = min(rows, r0 + rpb);
  constexpr int kU = 4;  // rows in flight per thread
  for (int rb = r0; rb < r1; rb += kU) {
    typename Chunk<T>::Raw rd[kU], rh[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (rb + u < r1) {
        const int64_t off = (int64_t)(rb + u) * U + col;
        rd[u] = Chunk<T>::ld(dA1 + off);
        rh[u] = Chunk<T>::ld(h + off);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int r = rb + u;
      if (r < r1) {
        float d[8], x[8];
        Chunk<T>::unpack(rd[u], d);
        Chunk<T>::unpack(rh[u], x);
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] += bb[j];
        float m[8];
        keep_mul8((uint64_t)(g0 + (int64_t)r * ncU + ch), pk, m);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          d[j] = d[j] * m[j] * act_df<ACT>(x[j]);
          acc[j] += d[j];
        }
        Chunk<T>::store(dh + (int64_t)r * U + col, d);
      }
    }
  }
  float* out = partials + (int64_t)blockIdx.y * U + col;
  reinterpret_cast<float4*>(out)[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
  reinterpret_cast<float4*>(out)[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
}

cudaError_t launch_bad_bwd(int dtype, int B, int J, int U, const void* dA1, const void* h,
                           const float* b1, int act, const PhiloxKey& pk, int64_t batch_offset,
                           void* dh, float* db1, const ReduceWs& ws, cudaStream_t st) {
  const int rows = B * J;
  if (rows == 0) return cudaMemsetAsync(db1, 0, sizeof(float) * U, st);
  const int ncU = U / 8;
  const int64_t g0 = batch_offset * (int64_t)J * ncU;
  const int gx = (ncU + 127) / 128;
  int R = (16 * ws.num_sms + gx - 1) / gx;   // ~16 row blocks per SM (measured: 8 -> 16 -2 us at L, -6 us at Bb)
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
          (const __nv_bfloat16*)dA1, (const __nv_bfloat16*)h, b1, (__nv_bfloat16*)dh,
          ws.partials, rows, rpb, U, g0, pk);
    else
      bad_bwd_kernel<float, ACT><<<grid, 128, 0, st>>>((const float*)dA1, (const float*)h, b1,
                                                       (float*)dh, ws.partials, rows, rpb, U,
                                                       g0, pk);
  });
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return colsum_finish(ws, R, U, U, db1, nullptr, nullptr, st);
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

// Keep bytes (R27 layout: one byte per 8-element chunk, bit u = element u) of a whole dropout
// site of `nchunks` chunks starting at Philox chunk g0: four independent Philox calls per
// thread (one 32-bit word of bytes).  The layer launches it for the BAD site on a side stream
// beside the fused score kernel, whose last wave leaves SMs idle (R29); the Linear1
// + BAD epilogue then reads the bytes instead of running Philox.
__global__ void __launch_bounds__(1024) keep_bytes_kernel(uint32_t* __restrict__ out,
                                                         int64_t nwords, int64_t g0,
                                                         PhiloxKey pk) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nwords;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t w = 0;
    float m[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) w |= keep_byte_mul8((uint64_t)(g0 + 4 * i + j), pk, m) << (8 * j);
    out[i] = w;
  }
}

cudaError_t launch_keep_bytes(int64_t nchunks, int64_t g0, const PhiloxKey& pk, uint8_t* out,
                              cudaStream_t st, int max_ctas) {
  if (nchunks <= 0) return cudaSuccess;
  if (nchunks % 4 || ((uintptr_t)out & 3u)) return cudaErrorInvalidValue;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t nwords = nchunks / 4;
  // 1024-thread CTAs: with max_ctas (the SMs a persistent kernel beside it leaves free) one
  // per free SM, else up to two per SM
  int64_t grid = (nwords + 1023) / 1024;
  const int64_t cap = max_ctas > 0 ? max_ctas : 2 * sms;
  if (grid > cap) grid = cap;
  keep_bytes_kernel<<<(int)grid, 1024, 0, st>>>(reinterpret_cast<uint32_t*>(out), nwords, g0,
                                                pk);
  return cudaGetLastError();
}

}  // namespace enc

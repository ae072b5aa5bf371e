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
#include "tma.cuh"

namespace enc {

// ------------------------------------------------------------------ BDRLN forward
template <typename T, int CPL>
__global__ void __launch_bounds__(256) bdrln_fwd_kernel(
    const T* __restrict__ Y, const float* __restrict__ bias, const T* __restrict__ R,
    const float* __restrict__ gamma, const float* __restrict__ beta, T* __restrict__ out,
    T* __restrict__ xhat, float* __restrict__ rstd_out, int rows, int I, float eps, int64_t g0,
    PhiloxKey pk, uint8_t* __restrict__ kb_out, const uint8_t* __restrict__ kb_in) {
  using C = Chunk<T>;
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int nc = I >> 3;
  const int64_t base = (int64_t)row * I;
  // all loads of the row first (2*CPL 16/32-byte loads in flight per lane)
  typename C::Raw ry[CPL], rr[CPL];
#pragma unroll
  for (int i = 0; i < CPL; ++i) {
    const int ch = lane + 32 * i;
    if (ch < nc) {
      ry[i] = C::ld(Y + base + ch * 8);
      rr[i] = C::ld(R + base + ch * 8);
    }
  }
  float z[CPL][8];
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < CPL; ++i) {
    const int ch = lane + 32 * i;
    if (ch < nc) {
      float y[8], b[8];
      C::unpack(ry[i], y);
      C::unpack(rr[i], z[i]);
      load_f32x8(bias + ch * 8, b);
      float m[8];
      keep_mul8_io(g0, (int64_t)row * nc + ch, pk, kb_out, kb_in, m);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        z[i][j] = fmaf(y[j] + b[j], m[j], z[i][j]);
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
      C::store(out + base + ch * 8, o);
      C::store(xhat + base + ch * 8, xh);
    }
  }
  if (lane == 0) rstd_out[row] = rstd;
}

cudaError_t launch_bdrln_fwd(int dtype, int B, int J, int I, const void* Y, const float* bias,
                             const void* R, const float* gamma, const float* beta, float eps,
                             const PhiloxKey& pk, int64_t batch_offset, void* out, void* xhat,
                             float* rstd, cudaStream_t st, int variant, uint8_t* kb_out,
                             const uint8_t* kb_in) {
  const int rows = B * J;
  if (rows == 0) return cudaSuccess;
  if (variant != 1 && bdrln_rg_supported(I))
    return launch_bdrln_fwd_rg(dtype, B, J, I, Y, bias, R, gamma, beta, eps, pk, batch_offset,
                               out, xhat, rstd, st, variant, kb_out, kb_in);
  const int nc = I / 8;
  const int64_t g0 = batch_offset * (int64_t)J * nc;
  const int grid = (rows + 7) / 8;
  ENC_CPL_DISPATCH(nc, {
    if (dtype == 0)
      bdrln_fwd_kernel<__nv_bfloat16, CPL><<<grid, 256, 0, st>>>(
          (const __nv_bfloat16*)Y, bias, (const __nv_bfloat16*)R, gamma, beta,
          (__nv_bfloat16*)out, (__nv_bfloat16*)xhat, rstd, rows, I, eps, g0, pk, kb_out, kb_in);
    else
      bdrln_fwd_kernel<float, CPL><<<grid, 256, 0, st>>>(
          (const float*)Y, bias, (const float*)R, gamma, beta, (float*)out, (float*)xhat, rstd,
          rows, I, eps, g0, pk, kb_out, kb_in);
  });
  return cudaGetLastError();
}

// ------------------------------------------------------------------ BDRLN backward
// Persistent: one CTA of 8 warps per SM, warp w of CTA c takes rows c*8+w, +8G, ...
// Each warp streams its rows through a 2-stage shared-memory ring filled by the bulk-copy
// (TMA) engine -- the next row's dOut and xhat land while the current one is computed,
// so a warp keeps two rows in flight without spending registers on them (the registers
// hold the three column-sum accumulators instead).
constexpr int kLnBwdWarps = 8;
constexpr int kLnBwdMaxSmem = 200 * 1024;

template <typename T, int CPL>
__global__ void __launch_bounds__(kLnBwdWarps * 32, 1) bdrln_bwd_kernel(
    const T* __restrict__ dOut, const T* __restrict__ xhat, const float* __restrict__ rstd,
    const float* __restrict__ gamma, T* __restrict__ dz, T* __restrict__ dYpre,
    float* __restrict__ partials, int rows, int I, int64_t g0, PhiloxKey pk, int kLnBwdStages,
    const uint8_t* __restrict__ kb_in) {
  using C = Chunk<T>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nc = I >> 3;
  const uint32_t row_bytes = (uint32_t)I * sizeof(T);
  // layout: mbar[warp][stage] | union { ring [warp][stage][2 tensors][I] T,
  //                                      red [warp][3][I] float (after the row loop) }
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* bar = bars + warp * kLnBwdStages;
  unsigned char* body = smem_raw + 128;
  T* ring = reinterpret_cast<T*>(body) + (size_t)warp * kLnBwdStages * 2 * I;
  float* red = reinterpret_cast<float*>(body);

  const int stride = gridDim.x * kLnBwdWarps;
  const int first = blockIdx.x * kLnBwdWarps + warp;
  if (lane == 0) {
    for (int s = 0; s < kLnBwdStages; ++s) mbar_init(&bar[s], 1);  // (1 or 2 stages)
    fence_mbar_init();
    for (int s = 0; s < kLnBwdStages; ++s) {
      const int r = first + s * stride;
      if (r < rows) {
        mbar_arrive_expect_tx(&bar[s], 2 * row_bytes);
        bulk_g2s(ring + (s * 2 + 0) * I, dOut + (int64_t)r * I, row_bytes, &bar[s]);
        bulk_g2s(ring + (s * 2 + 1) * I, xhat + (int64_t)r * I, row_bytes, &bar[s]);
      }
    }
  }
  __syncwarp();

  const float inv_n = 1.f / (float)I;
  float acc_g[CPL][8], acc_b[CPL][8], acc_d[CPL][8];
#pragma unroll
  for (int i = 0; i < CPL; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc_g[i][j] = acc_b[i][j] = acc_d[i][j] = 0.f;

  int k = 0;
  for (int row = first; row < rows; row += stride, ++k) {
    const int s = k % kLnBwdStages;
    mbar_wait(&bar[s], (uint32_t)(k / kLnBwdStages) & 1u);
    const T* sg = ring + (s * 2 + 0) * I;
    const T* sx = ring + (s * 2 + 1) * I;
    typename C::Raw rg[CPL], rx[CPL];
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
      const int ch = lane + 32 * i;
      if (ch < nc) {
        rg[i] = C::ld_smem(sg + ch * 8);
        rx[i] = C::ld_smem(sx + ch * 8);
      }
    }
    __syncwarp();
    if (lane == 0) {  // refill this stage with the row kStages ahead
      const int nr = row + kLnBwdStages * stride;
      if (nr < rows) {
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&bar[s], 2 * row_bytes);
        bulk_g2s(ring + (s * 2 + 0) * I, dOut + (int64_t)nr * I, row_bytes, &bar[s]);
        bulk_g2s(ring + (s * 2 + 1) * I, xhat + (int64_t)nr * I, row_bytes, &bar[s]);
      }
    }
    const float rs = __ldg(rstd + row);
    uint32_t kb[CPL];   // stored keep bytes (R27), loaded early with rstd
#pragma unroll
    for (int i = 0; i < CPL; ++i)
      kb[i] = (kb_in != nullptr && lane + 32 * i < nc)
                  ? (uint32_t)__ldg(kb_in + (int64_t)row * nc + lane + 32 * i)
                  : 0u;
    const int64_t base = (int64_t)row * I;
    float go[CPL][8], xh[CPL][8];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
      const int ch = lane + 32 * i;
      if (ch < nc) {
        float gm[8];
        C::unpack(rg[i], go[i]);
        C::unpack(rx[i], xh[i]);
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
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
      const int ch = lane + 32 * i;
      if (ch < nc) {
        float d[8], y[8], m[8];
        if (kb_in != nullptr)
          mul8_from_byte(kb[i], pk.scale, m);
        else
          keep_mul8((uint64_t)(g0 + (int64_t)row * nc + ch), pk, m);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          d[j] = rs * (go[i][j] - mg - xh[i][j] * mgx);
          y[j] = d[j] * m[j];
          acc_d[i][j] += y[j];
        }
        C::store(dz + base + ch * 8, d);
        C::store(dYpre + base + ch * 8, y);
      }
    }
  }
  // CTA reduction in a fixed order: every warp stores its three column-sum vectors to its
  // own slice (no read-modify-write chains), then each thread adds the 8 slices of its
  // columns in warp order.  The ring is dead by now (all its bulk copies were consumed).
  __syncthreads();
  float* mine = red + (size_t)warp * 3 * I;
#pragma unroll
  for (int i = 0; i < CPL; ++i) {
    const int ch = lane + 32 * i;
    if (ch < nc) {
      float4* d0 = reinterpret_cast<float4*>(mine + ch * 8);
      float4* d1 = reinterpret_cast<float4*>(mine + I + ch * 8);
      float4* d2 = reinterpret_cast<float4*>(mine + 2 * I + ch * 8);
      d0[0] = make_float4(acc_g[i][0], acc_g[i][1], acc_g[i][2], acc_g[i][3]);
      d0[1] = make_float4(acc_g[i][4], acc_g[i][5], acc_g[i][6], acc_g[i][7]);
      d1[0] = make_float4(acc_b[i][0], acc_b[i][1], acc_b[i][2], acc_b[i][3]);
      d1[1] = make_float4(acc_b[i][4], acc_b[i][5], acc_b[i][6], acc_b[i][7]);
      d2[0] = make_float4(acc_d[i][0], acc_d[i][1], acc_d[i][2], acc_d[i][3]);
      d2[1] = make_float4(acc_d[i][4], acc_d[i][5], acc_d[i][6], acc_d[i][7]);
    }
  }
  __syncthreads();
  float* out = partials + (int64_t)blockIdx.x * 3 * I;
  for (int c = threadIdx.x; c < 3 * I; c += blockDim.x) {
    float s = red[c];
#pragma unroll
    for (int w = 1; w < kLnBwdWarps; ++w) s += red[(size_t)w * 3 * I + c];
    out[c] = s;
  }
}

static size_t bdrln_bwd_smem(int I, size_t es, int stages) {
  const size_t ring = (size_t)kLnBwdWarps * stages * 2 * I * es;
  const size_t red = (size_t)kLnBwdWarps * 3 * I * sizeof(float);
  return 128 + (ring > red ? ring : red);
}

// 2-stage ring when it fits, else 1 stage; rows up to 2048 elements (8 chunks per lane)
static int bdrln_bwd_stages(int I, int dtype) {
  const size_t es = dtype == 0 ? 2 : 4;
  if (bdrln_bwd_smem(I, es, 2) <= kLnBwdMaxSmem) return 2;
  if (bdrln_bwd_smem(I, es, 1) <= kLnBwdMaxSmem) return 1;
  return 0;
}

bool bdrln_bwd_supported(int I, int dtype) {
  return rowop_supported(I) && I <= 2048 && bdrln_bwd_stages(I, dtype) > 0;
}

cudaError_t launch_bdrln_bwd(int dtype, int B, int J, int I, const void* dOut, const void* xhat,
                             const float* rstd, const float* gamma, const PhiloxKey& pk,
                             int64_t batch_offset, void* dz, void* dYpre, float* dgamma,
                             float* dbeta, float* dbias, const ReduceWs& ws, cudaStream_t st,
                             int variant, const uint8_t* kb_in) {
  const int rows = B * J;
  if (rows == 0) {
    cudaMemsetAsync(dgamma, 0, sizeof(float) * I, st);
    cudaMemsetAsync(dbeta, 0, sizeof(float) * I, st);
    return cudaMemsetAsync(dbias, 0, sizeof(float) * I, st);
  }
  if (variant != 1 && bdrln_rg_supported(I))
    return launch_bdrln_bwd_rg(dtype, B, J, I, dOut, xhat, rstd, gamma, pk, batch_offset, dz,
                               dYpre, dgamma, dbeta, dbias, ws, st, variant, kb_in);
  const int nc = I / 8;
  const int64_t g0 = batch_offset * (int64_t)J * nc;
  int G = (rows + kLnBwdWarps - 1) / kLnBwdWarps;
  if (G > ws.num_sms) G = ws.num_sms;
  const size_t cap = ws.cap_floats / (size_t)(3 * I);
  if ((size_t)G > cap) G = (int)cap;
  if (G < 1) G = 1;
  const int stages = bdrln_bwd_stages(I, dtype);
  if (stages == 0) return cudaErrorInvalidValue;
  const size_t smem = bdrln_bwd_smem(I, dtype == 0 ? 2 : 4, stages);
  ENC_CPL_DISPATCH8(nc, {
    {
      if (dtype == 0) {
        auto kern = bdrln_bwd_kernel<__nv_bfloat16, CPL>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<G, kLnBwdWarps * 32, smem, st>>>(
            (const __nv_bfloat16*)dOut, (const __nv_bfloat16*)xhat, rstd, gamma,
            (__nv_bfloat16*)dz, (__nv_bfloat16*)dYpre, ws.partials, rows, I, g0, pk, stages,
            kb_in);
      } else {
        auto kern = bdrln_bwd_kernel<float, CPL>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<G, kLnBwdWarps * 32, smem, st>>>((const float*)dOut, (const float*)xhat, rstd,
                                                gamma, (float*)dz, (float*)dYpre, ws.partials,
                                                rows, I, g0, pk, stages, kb_in);
      }
    }
  });
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return colsum_finish(ws, G, 3 * I, I, dgamma, dbeta, dbias, st);
}

// ------------------------------------------------------------------ column-sum finalize
// Block = 32 columns x 32 row-slices.  Thread (x, y) sums partial rows y, y+32, ... of its
// column (all loads issued first, ascending order), then the 32 slice sums are added in
// ascending y order: a fixed summation order, independent of timing.
constexpr int kFinY = 16;   // one resident wave of 512-thread blocks (32: 1.4 waves, +2 us)
constexpr int kFinMaxPer = 16;  // partial rows per slice handled with loads in flight

__global__ void __launch_bounds__(32 * kFinY) colsum_finalize_kernel(
    const float* __restrict__ partials, int R, int ncols, int nper, float* out0, float* out1,
    float* out2) {
  __shared__ float sm[kFinY][33];
  pdl_wait();   // the partials are the stream predecessor's outputs
  const int c = blockIdx.x * 32 + threadIdx.x;
  float s = 0.f;
  if (c < ncols) {
    for (int r0 = threadIdx.y; r0 < R; r0 += kFinY * kFinMaxPer) {
      // unconditional loads from clamped rows (issued back to back), masked afterwards
      float v[kFinMaxPer];
#pragma unroll
      for (int u = 0; u < kFinMaxPer; ++u) {
        const int r = min(r0 + u * kFinY, R - 1);
        v[u] = __ldg(partials + (int64_t)r * ncols + c);
      }
#pragma unroll
      for (int u = 0; u < kFinMaxPer; ++u) s += (r0 + u * kFinY < R) ? v[u] : 0.f;
    }
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
  return launch_k(PDL_FINAL, colsum_finalize_kernel, (ncols + 31) / 32, block, 0, st, partials, R, ncols,
                  nper, out0, out1, out2);
}

cudaError_t colsum_finish(const ReduceWs& ws, int R, int ncols, int nper, float* out0,
                          float* out1, float* out2, cudaStream_t st) {
  if (ws.defer != nullptr) {
    ColsumJob& j = *ws.defer;
    j.partials = ws.partials;
    j.R = R;
    j.ncols = ncols;
    j.nper = nper;
    j.out0 = out0;
    j.out1 = out1;
    j.out2 = out2;
    return cudaSuccess;
  }
  return launch_colsum_finalize(ws.partials, R, ncols, nper, out0, out1, out2, st);
}

struct ColsumJobs4 {
  ColsumJob j[4];
  int first_block[5];   // block ranges per job
};

__global__ void __launch_bounds__(32 * kFinY) colsum_finalize_jobs_kernel(ColsumJobs4 js) {
  __shared__ float sm[kFinY][33];
  pdl_wait();
  int k = 0;
  while (k < 3 && (int)blockIdx.x >= js.first_block[k + 1]) ++k;
  const ColsumJob& jb = js.j[k];
  const int c = ((int)blockIdx.x - js.first_block[k]) * 32 + threadIdx.x;
  float s = 0.f;
  if (c < jb.ncols) {
    for (int r0 = threadIdx.y; r0 < jb.R; r0 += kFinY * kFinMaxPer) {
      float v[kFinMaxPer];
#pragma unroll
      for (int u = 0; u < kFinMaxPer; ++u) {
        const int r = min(r0 + u * kFinY, jb.R - 1);
        v[u] = __ldg(jb.partials + (int64_t)r * jb.ncols + c);
      }
#pragma unroll
      for (int u = 0; u < kFinMaxPer; ++u) s += (r0 + u * kFinY < jb.R) ? v[u] : 0.f;
    }
  }
  sm[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.y == 0 && c < jb.ncols) {
    float t = sm[0][threadIdx.x];
#pragma unroll
    for (int y = 1; y < kFinY; ++y) t += sm[y][threadIdx.x];
    const int q = c / jb.nper;
    const int jj = c - q * jb.nper;
    float* o = q == 0 ? jb.out0 : (q == 1 ? jb.out1 : jb.out2);
    o[jj] = t;
  }
}

cudaError_t launch_colsum_finalize_jobs(const ColsumJob* jobs, int n, cudaStream_t st) {
  if (n < 1 || n > 4) return cudaErrorInvalidValue;
  ColsumJobs4 js{};
  int nb = 0;
  for (int k = 0; k < 4; ++k) {
    js.first_block[k] = nb;
    if (k < n) {
      js.j[k] = jobs[k];
      nb += (jobs[k].ncols + 31) / 32;
    }
  }
  js.first_block[4] = nb;
  if (nb == 0) return cudaSuccess;
  dim3 block(32, kFinY);
  launch_k(PDL_FINAL, colsum_finalize_jobs_kernel, nb, block, 0, st, js);
  return cudaGetLastError();
}

}  // namespace enc

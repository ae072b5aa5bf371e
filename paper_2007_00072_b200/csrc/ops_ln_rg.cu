// Row-group BDRLN kernels (forward and backward) for I % 32 == 0, I <= 2048.
//
// A row of I elements is shared by a group of GW warps (GW = 2 at I = 1024, 3 when a third
// of the row is exactly one 8-element chunk per lane, I = 768, else 4; each warp owns a contiguous part of
// the columns, at most 2 chunks of 8 per lane), so a warp's per-row work is a quarter of
// the one-warp-per-row kernels in ops_ln.cu and four times as many rows are in flight per
// SM.  Persistent CTAs of 4 groups (512 threads); each group streams its rows through a
// 2- or 4-stage shared-memory ring filled by the bulk-copy (TMA) engine.  A lane always owns
// the same columns, so bias / gamma / beta are loaded into registers once.  The
// row statistics of the 4 quarters are combined through shared memory behind one named
// barrier per row (forward: Chan's parallel mean / M2 combination, backward: the two
// LayerNorm-gradient sums), always in quarter order, so results do not depend on timing.
// The backward accumulates dgamma / dbeta / dbias column sums in registers (24 per
// thread), reduces them over the 4 groups in fixed order and writes one partial row per CTA
// for launch_colsum_finalize.
#include <math.h>

#include "kernels.h"
#include "tma.cuh"

namespace enc {
namespace {

constexpr int kGroups = 4;              // row groups per CTA (NG of the default variants)
constexpr int kWideGroups = 8;          // NG of the wide variant: 8 groups x GW warps per CTA
constexpr int kGWarps = 4;              // most warps per row group (header sizing)
constexpr int kRgMaxStages = 4;

template <int GW>
__device__ __forceinline__ void gbar(int group) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + group), "r"(GW * 32) : "memory");
}

// shared layout: mbar[group][stage] (256 B) | red[group][stage][GW] float4 |
// ring[group][stage][ntens][I] T | (bwd, after the loop) colsum[group][3][I] float
constexpr int kRgHdr = 256 + kWideGroups * kRgMaxStages * kGWarps * 16;

template <typename T, int NT, int STG>
__device__ __forceinline__ T* ring_row(unsigned char* smem, int I, int g, int s, int t) {
  return reinterpret_cast<T*>(smem + kRgHdr) + (((size_t)g * STG + s) * NT + t) * I;
}

// ------------------------------------------------------------------ forward
template <typename T, int CPW, int STG, int GW, int NG = kGroups>
__global__ void __launch_bounds__(NG * GW * 32, NG * GW * 32 > 512 ? 1 : (CPW == 1 ? 2 : 1))
bdrln_fwd_rg_kernel(
    const T* __restrict__ Y, const float* __restrict__ bias, const T* __restrict__ R,
    const float* __restrict__ gamma, const float* __restrict__ beta, T* __restrict__ out,
    T* __restrict__ xhat, float* __restrict__ rstd_out, int rows, int I, float eps, int64_t g0,
    PhiloxKey pk, uint8_t* __restrict__ kb_out, const uint8_t* __restrict__ kb_in) {
  using C = Chunk<T>;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = warp / GW, w = warp % GW;
  const int nc = I >> 3, ncq = nc / GW;          // chunks per row, per quarter
  const uint32_t row_bytes = (uint32_t)I * sizeof(T);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem) + g * STG;
  float4* red = reinterpret_cast<float4*>(smem + 256) + (size_t)g * STG * GW;
  const int stride = gridDim.x * NG;
  const int first = blockIdx.x * NG + g;
  const bool leader = (w == 0 && lane == 0);
  // this lane's columns are the same for every row: parameters into registers once (before
  // pdl_wait: they are not written by the stream predecessor)
  float pb[CPW][8], pg[CPW][8], pe[CPW][8];
#pragma unroll
  for (int i = 0; i < CPW; ++i) {
    const int ch = w * ncq + min(lane + 32 * i, ncq - 1);
    load_f32x8(bias + ch * 8, pb[i]);
    load_f32x8(gamma + ch * 8, pg[i]);
    load_f32x8(beta + ch * 8, pe[i]);
  }
  if (leader) {
    for (int s = 0; s < STG; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  pdl_wait();
  if (leader) {
    for (int s = 0; s < STG; ++s) {
      const int r = first + s * stride;
      if (r < rows) {
        mbar_arrive_expect_tx(&bar[s], 2 * row_bytes);
        bulk_g2s(ring_row<T, 2, STG>(smem, I, g, s, 0), Y + (int64_t)r * I, row_bytes, &bar[s]);
        bulk_g2s(ring_row<T, 2, STG>(smem, I, g, s, 1), R + (int64_t)r * I, row_bytes, &bar[s]);
      }
    }
  }
  gbar<GW>(g);
  int k = 0;
  for (int row = first; row < rows; row += stride, ++k) {
    const int s = k % STG;
    uint32_t kb[CPW];   // given keep bytes (R31), loaded before the row's data wait
#pragma unroll
    for (int i = 0; i < CPW; ++i)
      kb[i] = (kb_in != nullptr && lane + 32 * i < ncq)
                  ? (uint32_t)__ldg(kb_in + (int64_t)row * nc + w * ncq + lane + 32 * i)
                  : 0u;
    mbar_wait(&bar[s], (uint32_t)(k / STG) & 1u);
    const T* sy = ring_row<T, 2, STG>(smem, I, g, s, 0);
    const T* sr = ring_row<T, 2, STG>(smem, I, g, s, 1);
    float z[CPW][8];
    float lsum = 0.f;
#pragma unroll
    for (int i = 0; i < CPW; ++i) {
      const int cq = lane + 32 * i;
      if (cq < ncq) {
        const int ch = w * ncq + cq;
        float y[8], m[8];
        C::unpack(C::ld_smem(sy + ch * 8), y);
        C::unpack(C::ld_smem(sr + ch * 8), z[i]);
        if (kb_in != nullptr)
          mul8_from_byte(kb[i], pk.scale, m);
        else
          keep_mul8_io(g0, (int64_t)row * nc + ch, pk, kb_out, nullptr, m);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          z[i][j] = fmaf(y[j] + pb[i][j], m[j], z[i][j]);
          lsum += z[i][j];
        }
      }
    }
    // quarter mean and M2 (two passes over registers), then Chan's combination
    const float qn = (float)(ncq * 8);
    const float qmean = warp_sum(lsum) / qn;
    float m2 = 0.f;
#pragma unroll
    for (int i = 0; i < CPW; ++i) {
      if (lane + 32 * i < ncq) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float d = z[i][j] - qmean;
          m2 = fmaf(d, d, m2);
        }
      }
    }
    m2 = warp_sum(m2);
    if (lane == 0) red[s * GW + w] = make_float4(qmean, m2, 0.f, 0.f);
    gbar<GW>(g);   // quarter stats visible; every warp of the group has read this ring stage
    if (leader) {
      const int nr = row + STG * stride;
      if (nr < rows) {
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&bar[s], 2 * row_bytes);
        bulk_g2s(ring_row<T, 2, STG>(smem, I, g, s, 0), Y + (int64_t)nr * I, row_bytes, &bar[s]);
        bulk_g2s(ring_row<T, 2, STG>(smem, I, g, s, 1), R + (int64_t)nr * I, row_bytes, &bar[s]);
      }
    }
    float mean = 0.f;
#pragma unroll
    for (int q = 0; q < GW; ++q) mean += red[s * GW + q].x;
    mean *= 1.f / GW;
    float M2 = 0.f;
#pragma unroll
    for (int q = 0; q < GW; ++q) {
      const float4 st = red[s * GW + q];
      const float d = st.x - mean;
      M2 += st.y + qn * d * d;
    }
    const float rstd = rsqrtf(M2 / (float)I + eps);
    const int64_t base = (int64_t)row * I;
#pragma unroll
    for (int i = 0; i < CPW; ++i) {
      const int cq = lane + 32 * i;
      if (cq < ncq) {
        const int ch = w * ncq + cq;
        float xh[8], o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          xh[j] = (z[i][j] - mean) * rstd;
          o[j] = fmaf(pg[i][j], xh[j], pe[i][j]);
        }
        C::store(out + base + ch * 8, o);
        C::store(xhat + base + ch * 8, xh);
      }
    }
    if (leader) rstd_out[row] = rstd;
  }
}

// ------------------------------------------------------------------ backward
template <typename T, int CPW, int STG, int GW, int NG = kGroups>
__global__ void __launch_bounds__(NG * GW * 32, NG * GW * 32 > 512 ? 1 : (CPW == 1 ? 2 : 1))
bdrln_bwd_rg_kernel(
    const T* __restrict__ dOut, const T* __restrict__ xhat, const float* __restrict__ rstd,
    const float* __restrict__ gamma, T* __restrict__ dz, T* __restrict__ dYpre,
    float* __restrict__ partials, int rows, int I, int64_t g0, PhiloxKey pk,
    const uint8_t* __restrict__ kb_in) {
  using C = Chunk<T>;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = warp / GW, w = warp % GW;
  const int nc = I >> 3, ncq = nc / GW;
  const uint32_t row_bytes = (uint32_t)I * sizeof(T);
  const float inv_n = 1.f / (float)I;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem) + g * STG;
  float4* red = reinterpret_cast<float4*>(smem + 256) + (size_t)g * STG * GW;
  const int stride = gridDim.x * NG;
  const int first = blockIdx.x * NG + g;
  const bool leader = (w == 0 && lane == 0);
  if (leader) {
    for (int s = 0; s < STG; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  pdl_wait();   // dOut is the stream predecessor's output
  if (leader) {
    for (int s = 0; s < STG; ++s) {
      const int r = first + s * stride;
      if (r < rows) {
        mbar_arrive_expect_tx(&bar[s], 2 * row_bytes);
        bulk_g2s(ring_row<T, 2, STG>(smem, I, g, s, 0), dOut + (int64_t)r * I, row_bytes, &bar[s]);
        bulk_g2s(ring_row<T, 2, STG>(smem, I, g, s, 1), xhat + (int64_t)r * I, row_bytes, &bar[s]);
      }
    }
  }
  gbar<GW>(g);
  float acc_g[CPW][8], acc_b[CPW][8], acc_d[CPW][8];
#pragma unroll
  for (int i = 0; i < CPW; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc_g[i][j] = acc_b[i][j] = acc_d[i][j] = 0.f;
  int k = 0;
  for (int row = first; row < rows; row += stride, ++k) {
    const int s = k % STG;
    const float rs = __ldg(rstd + row);   // issued early: used after the row reduction
    uint32_t kb[CPW];                     // stored keep bytes (R27), issued early as well
#pragma unroll
    for (int i = 0; i < CPW; ++i)
      kb[i] = (kb_in != nullptr && lane + 32 * i < ncq)
                  ? (uint32_t)__ldg(kb_in + (int64_t)row * nc + w * ncq + lane + 32 * i)
                  : 0u;
    mbar_wait(&bar[s], (uint32_t)(k / STG) & 1u);
    const T* sg = ring_row<T, 2, STG>(smem, I, g, s, 0);
    const T* sx = ring_row<T, 2, STG>(smem, I, g, s, 1);
    float go[CPW][8], xh[CPW][8];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < CPW; ++i) {
      const int cq = lane + 32 * i;
      if (cq < ncq) {
        const int ch = w * ncq + cq;
        float gm[8];   // (gamma per row from L1: 24 accumulators already hold registers)
        C::unpack(C::ld_smem(sg + ch * 8), go[i]);
        C::unpack(C::ld_smem(sx + ch * 8), xh[i]);
        load_f32x8(gamma + ch * 8, gm);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          acc_g[i][j] = fmaf(go[i][j], xh[i][j], acc_g[i][j]);
          acc_b[i][j] += go[i][j];
          go[i][j] *= gm[j];
          s1 += go[i][j];
          s2 = fmaf(go[i][j], xh[i][j], s2);
        }
      }
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) red[s * GW + w] = make_float4(s1, s2, 0.f, 0.f);
    gbar<GW>(g);
    if (leader) {
      const int nr = row + STG * stride;
      if (nr < rows) {
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&bar[s], 2 * row_bytes);
        bulk_g2s(ring_row<T, 2, STG>(smem, I, g, s, 0), dOut + (int64_t)nr * I, row_bytes, &bar[s]);
        bulk_g2s(ring_row<T, 2, STG>(smem, I, g, s, 1), xhat + (int64_t)nr * I, row_bytes, &bar[s]);
      }
    }
    float t1 = 0.f, t2 = 0.f;
#pragma unroll
    for (int q = 0; q < GW; ++q) {
      const float4 st = red[s * GW + q];
      t1 += st.x;
      t2 += st.y;
    }
    const float mg = t1 * inv_n, mgx = t2 * inv_n;
    const int64_t base = (int64_t)row * I;
#pragma unroll
    for (int i = 0; i < CPW; ++i) {
      const int cq = lane + 32 * i;
      if (cq < ncq) {
        const int ch = w * ncq + cq;
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
  // column sums: each warp owns a column quarter; add the 4 groups in fixed order
  __syncthreads();   // ring is dead (all its bulk copies were consumed)
  float* colsum = reinterpret_cast<float*>(smem + kRgHdr);   // [group][3][I]
  float* mine = colsum + (size_t)g * 3 * I;
#pragma unroll
  for (int i = 0; i < CPW; ++i) {
    const int cq = lane + 32 * i;
    if (cq < ncq) {
      const int c0 = (w * ncq + cq) * 8;
#pragma unroll
      for (int j = 0; j < 8; j += 4) {
        *reinterpret_cast<float4*>(mine + c0 + j) =
            make_float4(acc_g[i][j], acc_g[i][j + 1], acc_g[i][j + 2], acc_g[i][j + 3]);
        *reinterpret_cast<float4*>(mine + I + c0 + j) =
            make_float4(acc_b[i][j], acc_b[i][j + 1], acc_b[i][j + 2], acc_b[i][j + 3]);
        *reinterpret_cast<float4*>(mine + 2 * I + c0 + j) =
            make_float4(acc_d[i][j], acc_d[i][j + 1], acc_d[i][j + 2], acc_d[i][j + 3]);
      }
    }
  }
  __syncthreads();
  float* outp = partials + (int64_t)blockIdx.x * 3 * I;
  for (int c = threadIdx.x; c < 3 * I; c += (NG * GW * 32)) {
    float v = colsum[c];
#pragma unroll
    for (int q = 1; q < NG; ++q) v += colsum[(size_t)q * 3 * I + c];
    outp[c] = v;
  }
}

// ring depth: 4 stages when the ring stays within ~96 KB (two CTAs per SM; the wide
// variant, one CTA per SM: 160 KB), else 2
int rg_stages(int I, size_t es, int ng = kGroups) {
  const size_t cap = ng == kWideGroups ? 160 * 1024 : 96 * 1024;
  return (size_t)ng * 4 * 2 * I * es <= cap ? 4 : 2;
}

size_t rg_smem(int I, size_t es, bool bwd, int ng = kGroups) {
  const size_t ring = (size_t)ng * rg_stages(I, es, ng) * 2 * I * es;
  const size_t cols = bwd ? (size_t)ng * 3 * I * sizeof(float) : 0;
  return kRgHdr + (ring > cols ? ring : cols);
}

// persistent grid: as many CTAs as can be resident (occupancy query), at most one group
// per row
template <typename Kern>
int rg_grid(Kern kern, int rows, size_t smem, int threads, int ng = kGroups) {
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  if (per_sm < 1) per_sm = 1;
  int G = (rows + ng - 1) / ng;
  if (G > per_sm * sms) G = per_sm * sms;
  return G < 1 ? 1 : G;
}

}  // namespace

// quarters of whole chunks, at most 2 chunks per lane
bool bdrln_rg_supported(int I) { return I % 32 == 0 && I <= 2048; }

#define ENC_CPW_DISPATCH(ncq, ...)                             \
  do {                                                         \
    if ((ncq) <= 32) { constexpr int CPW = 1; __VA_ARGS__; }   \
    else { constexpr int CPW = 2; __VA_ARGS__; }               \
  } while (0)
// warps per row: 2 at I = 1024 (two chunks per lane; in-graph A/B against 4 warps: BDRLN-bwd
// 17.0 -> 14.8 us, the step -4.6 us), 3 when a third of the row is exactly one chunk per lane
// (I = 768: BERT-base), else 4 -- no idle lanes where the row allows it
static int rg_gw(int nc) {
  if (nc == 128) return 2;   // I = 1024: two warps x two chunks per lane (measured faster than 4 x 1)
  return (nc % 96 == 0 && nc / 3 <= 64) ? 3 : 4;
}
// a requested warps-per-row count is usable when it splits the row's chunks evenly into at
// most two chunks per lane (the compiled CPW variants)
static bool rg_gw_valid(int nc, int gw) {
  return (gw == 2 || gw == 3 || gw == 4) && nc % gw == 0 && nc / gw <= 64;
}
#define ENC_GW_DISPATCH(gw, ...)                               \
  do {                                                         \
    if ((gw) == 2) { constexpr int GW = 2; __VA_ARGS__; }      \
    else if ((gw) == 3) { constexpr int GW = 3; __VA_ARGS__; } \
    else { constexpr int GW = 4; __VA_ARGS__; }                \
  } while (0)
#define ENC_STG_DISPATCH(stg, ...)                             \
  do {                                                         \
    if ((stg) == 4) { constexpr int STG = 4; __VA_ARGS__; }    \
    else { constexpr int STG = 2; __VA_ARGS__; }               \
  } while (0)
// wide variant (ENC_OPT_BDRLN_VARIANT 5): 8 row groups of nc/32 warps (one chunk per lane),
// up to 1024 threads in one CTA per SM -- twice the resident warps of the default for the
// same one partial row per CTA in the backward
static bool rg_wide_valid(int nc) { return nc % 32 == 0 && nc / 32 >= 2 && nc / 32 <= 4; }

cudaError_t launch_bdrln_fwd_rg(int dtype, int B, int J, int I, const void* Y, const float* bias,
                                const void* R, const float* gamma, const float* beta, float eps,
                                const PhiloxKey& pk, int64_t batch_offset, void* out, void* xhat,
                                float* rstd, cudaStream_t st, int gw_req, uint8_t* kb_out,
                                const uint8_t* kb_in) {
  const int rows = B * J;
  const int nc = I / 8;
  const int64_t g0 = batch_offset * (int64_t)J * nc;
  if (gw_req == 5 && rg_wide_valid(nc)) {
    constexpr int NG = kWideGroups;
    const size_t smem = rg_smem(I, dtype == 0 ? 2 : 4, false, NG);
    const int stg = rg_stages(I, dtype == 0 ? 2 : 4, NG);
    ENC_GW_DISPATCH(nc / 32, ENC_STG_DISPATCH(stg, {
      constexpr int thr = NG * GW * 32;
      if (dtype == 0) {
        auto kern = bdrln_fwd_rg_kernel<__nv_bfloat16, 1, STG, GW, NG>;
        launch_k(PDL_LN, kern, rg_grid(kern, rows, smem, thr, NG), thr, smem, st,
                 (const __nv_bfloat16*)Y, bias, (const __nv_bfloat16*)R, gamma, beta,
                 (__nv_bfloat16*)out, (__nv_bfloat16*)xhat, rstd, rows, I, eps, g0, pk, kb_out,
                 kb_in);
      } else {
        auto kern = bdrln_fwd_rg_kernel<float, 1, STG, GW, NG>;
        kern<<<rg_grid(kern, rows, smem, thr, NG), thr, smem, st>>>(
            (const float*)Y, bias, (const float*)R, gamma, beta, (float*)out, (float*)xhat,
            rstd, rows, I, eps, g0, pk, kb_out, kb_in);
      }
    }));
    return cudaGetLastError();
  }
  const size_t smem = rg_smem(I, dtype == 0 ? 2 : 4, false);
  const int stg = rg_stages(I, dtype == 0 ? 2 : 4);
  const int gw = rg_gw_valid(nc, gw_req) ? gw_req : rg_gw(nc);
  ENC_GW_DISPATCH(gw, ENC_CPW_DISPATCH(nc / gw, ENC_STG_DISPATCH(stg, {
    constexpr int thr = kGroups * GW * 32;
    if (dtype == 0) {
      auto kern = bdrln_fwd_rg_kernel<__nv_bfloat16, CPW, STG, GW>;
      launch_k(PDL_LN, kern, rg_grid(kern, rows, smem, thr), thr, smem, st,
               (const __nv_bfloat16*)Y, bias, (const __nv_bfloat16*)R, gamma, beta,
               (__nv_bfloat16*)out, (__nv_bfloat16*)xhat, rstd, rows, I, eps, g0, pk, kb_out,
               kb_in);
    } else {
      auto kern = bdrln_fwd_rg_kernel<float, CPW, STG, GW>;
      kern<<<rg_grid(kern, rows, smem, thr), thr, smem, st>>>(
          (const float*)Y, bias, (const float*)R, gamma, beta, (float*)out, (float*)xhat, rstd,
          rows, I, eps, g0, pk, kb_out, kb_in);
    }
  })));
  return cudaGetLastError();
}

cudaError_t launch_bdrln_bwd_rg(int dtype, int B, int J, int I, const void* dOut,
                                const void* xhat, const float* rstd, const float* gamma,
                                const PhiloxKey& pk, int64_t batch_offset, void* dz,
                                void* dYpre, float* dgamma, float* dbeta, float* dbias,
                                const ReduceWs& ws, cudaStream_t st, int gw_req,
                                const uint8_t* kb_in) {
  const int rows = B * J;
  const int nc = I / 8;
  const int64_t g0 = batch_offset * (int64_t)J * nc;
  const int cap = (int)(ws.cap_floats / (size_t)(3 * I));
  int G = 1;
  if (gw_req == 5 && rg_wide_valid(nc)) {
    constexpr int NG = kWideGroups;
    const size_t smem = rg_smem(I, dtype == 0 ? 2 : 4, true, NG);
    const int stg = rg_stages(I, dtype == 0 ? 2 : 4, NG);
    ENC_GW_DISPATCH(nc / 32, ENC_STG_DISPATCH(stg, {
      constexpr int thr = NG * GW * 32;
      if (dtype == 0) {
        auto kern = bdrln_bwd_rg_kernel<__nv_bfloat16, 1, STG, GW, NG>;
        G = rg_grid(kern, rows, smem, thr, NG);
        if (G > cap) G = cap;
        launch_k(PDL_LN, kern, G, thr, smem, st, (const __nv_bfloat16*)dOut,
                 (const __nv_bfloat16*)xhat, rstd, gamma, (__nv_bfloat16*)dz,
                 (__nv_bfloat16*)dYpre, ws.partials, rows, I, g0, pk, kb_in);
      } else {
        auto kern = bdrln_bwd_rg_kernel<float, 1, STG, GW, NG>;
        G = rg_grid(kern, rows, smem, thr, NG);
        if (G > cap) G = cap;
        kern<<<G, thr, smem, st>>>((const float*)dOut, (const float*)xhat, rstd, gamma,
                                   (float*)dz, (float*)dYpre, ws.partials, rows, I, g0, pk,
                                   kb_in);
      }
    }));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return colsum_finish(ws, G, 3 * I, I, dgamma, dbeta, dbias, st);
  }
  const size_t smem = rg_smem(I, dtype == 0 ? 2 : 4, true);
  const int stg = rg_stages(I, dtype == 0 ? 2 : 4);
  const int gw = rg_gw_valid(nc, gw_req) ? gw_req : rg_gw(nc);
  ENC_GW_DISPATCH(gw, ENC_CPW_DISPATCH(nc / gw, ENC_STG_DISPATCH(stg, {
    constexpr int thr = kGroups * GW * 32;
    if (dtype == 0) {
      auto kern = bdrln_bwd_rg_kernel<__nv_bfloat16, CPW, STG, GW>;
      G = rg_grid(kern, rows, smem, thr);
      if (G > cap) G = cap;
      launch_k(PDL_LN, kern, G, thr, smem, st, (const __nv_bfloat16*)dOut,
               (const __nv_bfloat16*)xhat, rstd, gamma, (__nv_bfloat16*)dz,
               (__nv_bfloat16*)dYpre, ws.partials, rows, I, g0, pk, kb_in);
    } else {
      auto kern = bdrln_bwd_rg_kernel<float, CPW, STG, GW>;
      G = rg_grid(kern, rows, smem, thr);
      if (G > cap) G = cap;
      kern<<<G, thr, smem, st>>>((const float*)dOut, (const float*)xhat, rstd, gamma,
                                 (float*)dz, (float*)dYpre, ws.partials, rows, I, g0, pk, kb_in);
    }
  })));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return colsum_finish(ws, G, 3 * I, I, dgamma, dbeta, dbias, st);
}

}  // namespace enc

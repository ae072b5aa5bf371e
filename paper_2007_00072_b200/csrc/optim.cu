// AdamW parameter update (decoupled weight decay) for the encoder stack's training step:
// one launch updates a layer's flat fp32 master parameters, first and second moments from
// its flat fp32 gradient buffer and writes the model copies the layer reads (bf16 or fp32
// weights, fp32 biases / gamma / beta) through a segment table.  The optimizer is outside
// the paper's method (the paper times encoder layers); the update is
// the AdamW definition (Loshchilov & Hutter; torch.optim.AdamW):
//   m = b1 m + (1 - b1) g,  v = b2 v + (1 - b2) g^2,
//   p = p (1 - lr wd) - lr (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps).
// Element-wise and HBM-bound: 16 B read + 12 B written per element of master / m / v / g,
// plus the model copy (2 or 4 B).  Four elements per thread (float4), grid-stride.
#include "kernels.h"

namespace enc {
namespace {

struct OptSegs {
  int count;
  OptSeg s[kOptMaxSegs];
};

__global__ void __launch_bounds__(256) adamw_kernel(float* __restrict__ master,
                                                    float* __restrict__ m1,
                                                    float* __restrict__ m2,
                                                    const float* __restrict__ g, int64_t n4,
                                                    OptSegs segs, float b1, float omb1,
                                                    float b2, float omb2, float eps,
                                                    float decay, float lr_bc1, float rsbc2,
                                                    float gscale) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 p = reinterpret_cast<float4*>(master)[i];
    float4 a = reinterpret_cast<float4*>(m1)[i];
    float4 b = reinterpret_cast<float4*>(m2)[i];
    const float4 gg = reinterpret_cast<const float4*>(g)[i];
    float pv[4] = {p.x, p.y, p.z, p.w}, av[4] = {a.x, a.y, a.z, a.w};
    float bv[4] = {b.x, b.y, b.z, b.w};
    const float gv[4] = {gg.x, gg.y, gg.z, gg.w};
    // the segment holding elements 4i .. 4i+3 (segments are 4-aligned): its model copy and
    // whether it takes weight decay
    const int64_t e = i * 4;
    int k = 0;
    while (k + 1 < segs.count && e >= segs.s[k + 1].begin) ++k;
    const OptSeg& sg = segs.s[k];
    const float dec = sg.no_decay ? 1.f : decay;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float gj = gv[j] * gscale;
      av[j] = fmaf(b1, av[j], omb1 * gj);
      bv[j] = fmaf(b2, bv[j], omb2 * gj * gj);
      const float denom = sqrtf(bv[j]) * rsbc2 + eps;   // sqrt(v / (1 - b2^t)) + eps
      pv[j] = pv[j] * dec - lr_bc1 * av[j] / denom;   // lr_bc1 = lr / (1 - b1^t)
    }
    reinterpret_cast<float4*>(master)[i] = make_float4(pv[0], pv[1], pv[2], pv[3]);
    reinterpret_cast<float4*>(m1)[i] = make_float4(av[0], av[1], av[2], av[3]);
    reinterpret_cast<float4*>(m2)[i] = make_float4(bv[0], bv[1], bv[2], bv[3]);
    const int64_t off = e - sg.begin;
    if (sg.dtype == 0) {
      uint2 u;
      u.x = Chunk<__nv_bfloat16>::pack2(pv[0], pv[1]);
      u.y = Chunk<__nv_bfloat16>::pack2(pv[2], pv[3]);
      reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(sg.out) + off)[0] = u;
    } else {
      reinterpret_cast<float4*>(static_cast<float*>(sg.out) + off)[0] =
          make_float4(pv[0], pv[1], pv[2], pv[3]);
    }
  }
}

}  // namespace

cudaError_t launch_adamw(int64_t n, float* master, float* m1, float* m2, const float* g,
                         const OptSeg* segs, int nseg, double lr, double b1, double b2,
                         double eps, double wd, int step, double gscale, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  OptSegs s{};
  s.count = nseg;
  for (int i = 0; i < nseg; ++i) s.s[i] = segs[i];
  // scalar coefficients formed in fp64 on the host, rounded once to fp32
  const double bc1 = 1.0 - pow(b1, (double)step);
  const double bc2 = 1.0 - pow(b2, (double)step);
  const int64_t n4 = n / 4;
  int64_t grid = (n4 + 255) / 256;
  if (grid > 148 * 8) grid = 148 * 8;
  adamw_kernel<<<(int)grid, 256, 0, st>>>(master, m1, m2, g, n4, s, (float)b1, (float)(1.0 - b1),
                                          (float)b2, (float)(1.0 - b2), (float)eps,
                                          (float)(1.0 - lr * wd), (float)(lr / bc1),
                                          (float)(1.0 / sqrt(bc2)), (float)gscale);
  return cudaGetLastError();
}

}  // namespace enc

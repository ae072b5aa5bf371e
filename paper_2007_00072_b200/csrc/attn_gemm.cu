// Hand-written tcgen05 batched contractions of multi-head attention (Table A.1 rows QK^T,
// Gamma and their dX1/dX2) for sm_100a.
//
// One CTA computes a 128 x BN tile of one (b, h) pair:
//   warp 0      TMA producer (one elected lane): 4-stage smem ring of A/B k-blocks
//   warp 1      TMEM allocator + MMA issuer (one elected lane): tcgen05.mma M=128, N=BN,
//               K=16 per instruction, fp32 accumulator in TMEM
//   warps 2-5   epilogue: tcgen05.ld 32 columns at a time -> bf16 -> global
// Operands are addressed through 4-D TMA tensor maps so the two-level (b, h) batch and the
// head-interleaved [B,J,H,P] layout of C / dC need no permute kernel and no pointer tables.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.h"
#include "tc_gemm.cuh"

namespace enc {

constexpr int kBM = 128;
constexpr int kBK = 64;       // one 128-byte swizzle row of bf16 along K
constexpr int kThreads = 192; // 6 warps

struct AttnGemmParams {
  int M, N, Kred, H;
  int a_mn, b_mn;            // operand majors (0 = K-major, 1 = MN-major)
  int a_rowdim, b_rowdim;    // tensor-map dim holding the row index (1 or 2); the other holds h
  int c_rowdim;
};

__device__ __forceinline__ void op_coords(int rowdim, int inner, int row, int h, int b, int* c) {
  c[0] = inner;
  if (rowdim == 1) {
    c[1] = row;
    c[2] = h;
  } else {
    c[1] = h;
    c[2] = row;
  }
  c[3] = b;
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1) attn_gemm_kernel(
    const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
    const __grid_constant__ CUtensorMap mapC, AttnGemmParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-B aligned operand ring (SWIZZLE_128B atoms), then barriers; after the last MMA the
  // ring is reused as the epilogue's TMA-store staging buffers
  unsigned char* base = tc::align1024(smem_raw);
  constexpr uint32_t kABytes = kBM * kBK * 2;
  constexpr uint32_t kBBytes = BN * kBK * 2;
  static_assert(STAGES * (kABytes + kBBytes) >= 4 * 2 * 4096, "staging must fit in the ring");
  unsigned char* sA = base;
  unsigned char* sB = base + STAGES * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * kBBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int bh = blockIdx.z;
  const int b = bh / p.H, h = bh - (bh / p.H) * p.H;
  const int m0 = blockIdx.y * kBM;
  const int n0 = blockIdx.x * BN;
  const int nk = p.Kred / kBK;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&mapA);
    tc::prefetch_tmap(&mapB);
    tc::prefetch_tmap(&mapC);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, BN < 32 ? 32 : BN);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        mbar_wait(&empty[s], ((kb / STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], kABytes + kBBytes);
        int c[4];
        const int k0 = kb * kBK;
        if (!p.a_mn) {
          op_coords(p.a_rowdim, k0, m0, h, b, c);
          tc::tma_load_4d(sA + s * kABytes, &mapA, &full[s], c[0], c[1], c[2], c[3]);
        } else {
#pragma unroll
          for (int blk = 0; blk < kBM / 64; ++blk) {
            op_coords(p.a_rowdim, m0 + 64 * blk, k0, h, b, c);
            tc::tma_load_4d(sA + s * kABytes + blk * 8192, &mapA, &full[s], c[0], c[1], c[2], c[3]);
          }
        }
        if (!p.b_mn) {
          op_coords(p.b_rowdim, k0, n0, h, b, c);
          tc::tma_load_4d(sB + s * kBBytes, &mapB, &full[s], c[0], c[1], c[2], c[3]);
        } else {
#pragma unroll
          for (int blk = 0; blk < BN / 64; ++blk) {
            op_coords(p.b_rowdim, n0 + 64 * blk, k0, h, b, c);
            tc::tma_load_4d(sB + s * kBBytes + blk * 8192, &mapB, &full[s], c[0], c[1], c[2], c[3]);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc = tc::instr_desc_bf16_f32(kBM, BN, p.a_mn, p.b_mn);
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&full[s], (kb / STAGES) & 1);
      tc::fence_after_sync();
      if (lane == 0) {
        const uint64_t ad0 = p.a_mn ? tc::smem_desc(smem_u32(sA + s * kABytes), 8192, 1024)
                                    : tc::smem_desc(smem_u32(sA + s * kABytes), 16, 1024);
        const uint64_t bd0 = p.b_mn ? tc::smem_desc(smem_u32(sB + s * kBBytes), 8192, 1024)
                                    : tc::smem_desc(smem_u32(sB + s * kBBytes), 16, 1024);
        const uint32_t astep = p.a_mn ? 2048 : 32, bstep = p.b_mn ? 2048 : 32;
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k)
          tc::mma_bf16(tmem, tc::desc_adv(ad0, k * astep), tc::desc_adv(bd0, k * bstep), idesc,
                       (kb | k) != 0);
        tc::mma_commit(&empty[s]);
        if (kb == nk - 1) tc::mma_commit(tmem_full);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogue
    // warp -> TMEM lane quarter q (rows m0+32q ..); per 64 columns: 2 x tcgen05.ld, pack to
    // bf16 into a 128-B-swizzled [32 x 64] staging tile, one TMA store per tile (double
    // buffered per warp)
    const int q = warp & 3;
    mbar_wait(tmem_full, 0);
    tc::fence_after_sync();
    unsigned char* stg = base + q * 2 * 4096;
#pragma unroll 1
    for (int c64 = 0; c64 < BN / 64; ++c64) {
      unsigned char* buf = stg + (c64 & 1) * 4096;
      if (c64 >= 2) {
        if (lane == 0) tc::bulk_wait_read<1>();
        __syncwarp();
      }
      float v[64];
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + c64 * 64;
      tc::tmem_ld32(taddr, v);
      tc::tmem_ld32(taddr + 32, v + 32);
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        uint4 u;
        u.x = Chunk<__nv_bfloat16>::pack2(v[8 * ch + 0], v[8 * ch + 1]);
        u.y = Chunk<__nv_bfloat16>::pack2(v[8 * ch + 2], v[8 * ch + 3]);
        u.z = Chunk<__nv_bfloat16>::pack2(v[8 * ch + 4], v[8 * ch + 5]);
        u.w = Chunk<__nv_bfloat16>::pack2(v[8 * ch + 6], v[8 * ch + 7]);
        *reinterpret_cast<uint4*>(buf + tc::sw128(lane, ch)) = u;
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        int c[4];
        op_coords(p.c_rowdim, n0 + c64 * 64, m0 + q * 32, h, b, c);
        tc::tma_store_4d(&mapC, buf, c[0], c[1], c[2], c[3]);
        tc::bulk_commit();
      }
    }
    if (lane == 0) tc::bulk_wait<0>();
    __syncwarp();
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, BN < 32 ? 32 : BN);
}

// ------------------------------------------------------------------ host side
namespace {
// 4-D bf16 tensor map: dims[0] innermost (contiguous), strides in elements for dims 1..3
bool make_map(CUtensorMap* m, const void* ptr, const uint64_t dims[4], const uint64_t strides[3],
              const uint32_t box[4]) {
  cuuint64_t gdim[4] = {dims[0], dims[1], dims[2], dims[3]};
  cuuint64_t gstride[3] = {strides[0] * 2, strides[1] * 2, strides[2] * 2};
  cuuint32_t bdim[4] = {box[0], box[1], box[2], box[3]};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = tmap_encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4,
                                      const_cast<void*>(ptr), gdim, gstride, bdim, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// operand layouts
enum Lay { BHJX = 0, BJHP = 1 };

// Map of a logical [B*H][rows][cols] operand (cols contiguous) with `lay`:
//  BHJX: physical [B][H][rows][cols];  BJHP: physical [B][rows][H][cols] (cols = P)
// box: `inner` x `rows_box` (rows along the row dim).
bool operand_map(CUtensorMap* m, const void* ptr, int lay, int B, int H, int rows, int cols,
                 int rows_box, int* rowdim) {
  uint64_t dims[4], strides[3];
  uint32_t box[4];
  if (lay == BHJX) {
    dims[0] = cols; dims[1] = rows; dims[2] = H; dims[3] = B;
    strides[0] = cols; strides[1] = (uint64_t)rows * cols; strides[2] = (uint64_t)H * rows * cols;
    box[0] = 64; box[1] = rows_box; box[2] = 1; box[3] = 1;
    *rowdim = 1;
  } else {
    dims[0] = cols; dims[1] = H; dims[2] = rows; dims[3] = B;
    strides[0] = cols; strides[1] = (uint64_t)H * cols; strides[2] = (uint64_t)rows * H * cols;
    box[0] = 64; box[1] = 1; box[2] = rows_box; box[3] = 1;
    *rowdim = 2;
  }
  return make_map(m, ptr, dims, strides, box);
}
}  // namespace

bool attn_gemm_supported(int J, int P) {
  return J % 128 == 0 && P == 64;
}

template <int BN, int STAGES>
static cudaError_t launch_tile(dim3 grid, const CUtensorMap& ma, const CUtensorMap& mb,
                               const CUtensorMap& mc, const AttnGemmParams& p, cudaStream_t st) {
  const size_t smem = 1024 + STAGES * (kBM * kBK * 2 + (size_t)BN * kBK * 2) + 256;
  cudaFuncSetAttribute(attn_gemm_kernel<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  attn_gemm_kernel<BN, STAGES><<<grid, kThreads, smem, st>>>(ma, mb, mc, p);
  return cudaGetLastError();
}

// which: 0 S=QK^T, 1 C=AV, 2 dA=dC V^T, 3 dV=A^T dC, 4 dQ=dS K, 5 dK=dS^T Q
// P-wide operands through map_pop (coordinates (p, h, row, b): row dim 2) with their row
// strides; [J x K] operands head-major [B,H,J,K] (row dim 1).
cudaError_t launch_attn_gemm(int which, int B, int H, int J, int P, const void* X, int64_t ldx,
                             const void* Y, int64_t ldy, void* Z, int64_t ldz, cudaStream_t st,
                             int Kkeys) {
  // J query rows, K key rows (self-attention: K = J; encoder-decoder attention: K keys of
  // the memory sequence)
  const int K = Kkeys > 0 ? Kkeys : J;
  if (J % kBM || K % kBM) return cudaErrorInvalidValue;
  AttnGemmParams p{};
  p.H = H;
  CUtensorMap ma, mb, mc;
  bool ok = true;
  int BN = 64;
  auto pop = [&](CUtensorMap* m, const void* ptr, int rows, int64_t ld, int box, int* rowdim) {
    *rowdim = 2;
    return map_pop(m, ptr, B, H, rows, P, ld, box);
  };
  switch (which) {
    case 0:  // S[J,K] = Q[J,P] K[K,P]^T : A K-major (Q rows), B K-major (K rows)
      p.M = J; p.N = K; p.Kred = P; BN = K % 256 == 0 ? 256 : 128;
      ok &= pop(&ma, X, J, ldx, kBM, &p.a_rowdim);
      ok &= pop(&mb, Y, K, ldy, BN, &p.b_rowdim);
      ok &= operand_map(&mc, Z, BHJX, B, H, J, K, 32, &p.c_rowdim);
      break;
    case 1:  // C[J,P] = A[J,K] V[K,P] : A K-major, B MN-major (V rows = K)
      p.M = J; p.N = P; p.Kred = K; BN = P; p.b_mn = 1;
      ok &= operand_map(&ma, X, BHJX, B, H, J, K, kBM, &p.a_rowdim);
      ok &= pop(&mb, Y, K, ldy, kBK, &p.b_rowdim);
      ok &= pop(&mc, Z, J, ldz, 32, &p.c_rowdim);
      break;
    case 2:  // dA[J,K] = dC[J,P] V[K,P]^T : dC K-major, V K-major
      p.M = J; p.N = K; p.Kred = P; BN = K % 256 == 0 ? 256 : 128;
      ok &= pop(&ma, X, J, ldx, kBM, &p.a_rowdim);
      ok &= pop(&mb, Y, K, ldy, BN, &p.b_rowdim);
      ok &= operand_map(&mc, Z, BHJX, B, H, J, K, 32, &p.c_rowdim);
      break;
    case 3:  // dV[K,P] = A[J,K]^T dC[J,P] : A MN-major (rows = J = Kred), dC MN-major
      p.M = K; p.N = P; p.Kred = J; BN = P; p.a_mn = 1; p.b_mn = 1;
      ok &= operand_map(&ma, X, BHJX, B, H, J, K, kBK, &p.a_rowdim);
      ok &= pop(&mb, Y, J, ldy, kBK, &p.b_rowdim);
      ok &= pop(&mc, Z, K, ldz, 32, &p.c_rowdim);
      break;
    case 4:  // dQ[J,P] = dS[J,K] K[K,P] : dS K-major, K MN-major
      p.M = J; p.N = P; p.Kred = K; BN = P; p.b_mn = 1;
      ok &= operand_map(&ma, X, BHJX, B, H, J, K, kBM, &p.a_rowdim);
      ok &= pop(&mb, Y, K, ldy, kBK, &p.b_rowdim);
      ok &= pop(&mc, Z, J, ldz, 32, &p.c_rowdim);
      break;
    case 5:  // dK[K,P] = dS[J,K]^T Q[J,P] : dS MN-major (rows = J), Q MN-major
      p.M = K; p.N = P; p.Kred = J; BN = P; p.a_mn = 1; p.b_mn = 1;
      ok &= operand_map(&ma, X, BHJX, B, H, J, K, kBK, &p.a_rowdim);
      ok &= pop(&mb, Y, J, ldy, kBK, &p.b_rowdim);
      ok &= pop(&mc, Z, K, ldz, 32, &p.c_rowdim);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  if (!ok) return cudaErrorInvalidValue;
  dim3 grid(p.N / BN, p.M / kBM, B * H);
  // Kred = P = 64 (one k-block): a single stage, so two CTAs fit per SM;
  // Kred = J: a 4-stage TMA ring
  if (BN == 256) return launch_tile<256, 1>(grid, ma, mb, mc, p, st);
  if (BN == 128) return launch_tile<128, 2>(grid, ma, mb, mc, p, st);
  if (BN == 64) return launch_tile<64, 4>(grid, ma, mb, mc, p, st);
  return cudaErrorInvalidValue;
}

}  // namespace enc

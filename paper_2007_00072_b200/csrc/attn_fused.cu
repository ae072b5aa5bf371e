// Fused attention-score kernels: a tcgen05 contraction whose epilogue is the paper's
// statistical-normalisation operator, so the score tensor never goes to HBM.
//
//  attn_qk_bsb   S = Q K^T (Table A.1 :551) -> BSB (`sm`, :552): P = softmax(scale*S + M),
//                A = dropout(P); writes P and A only.  Saves the S write + S read of the
//                unfused pair (2 x B*H*J*K*2 bytes = 134 MB at config L).
//  attn_da_bsbb  dA = dC V^T (:588) -> BSB-bwd (`bs`, :590): dP = dropout(dA),
//                dS = scale * P * (dP - sum_k dP*P); reads P, writes dS only.  Saves the dA
//                write + dA read (134 MB at config L).
//
// Tile = one (b, h) pair x 128 query rows x all K keys (K in {256, 512}): the fp32 score /
// gradient tile (128 x K) occupies K TMEM columns, so each row's softmax statistics are
// complete inside the CTA.  Persistent CTAs (one per SM) walk the tile list; warp roles:
//   warp 0      TMA producer: operands of the next tile as soon as the MMA released them
//               (and, bwd, the P tile of the next tile once its dS stores drained)
//   warp 1      TMEM owner + MMA issuer (one elected lane, N <= 256 per tcgen05.mma)
//   warps 2-17  epilogue: the 4 warps of TMEM lane quarter q each own a K/4-column slice of
//               rows 32q..32q+31; row statistics of the 4 slices are combined through
//               shared memory (named barrier per quarter); results leave through
//               128-B-swizzled staging tiles and TMA stores.
// Forward epilogue: pass 1 row max (no exponentials), pass 2 e = 2^(y - max) written back
// to TMEM + row sum (one MUFU.EX2 per element), pass 3 P = e / sum and A = dropout(P).
// Backward epilogue: pass 1 sum_k dropout(dA)*P (keep bits cached in shared memory), pass 2
// dS, staged in place of the P tile it was computed from.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "kernels.h"
#include "tc_gemm.cuh"

namespace enc {
namespace {

constexpr int kRows = 128;          // query rows per tile (MMA M)
constexpr int kEpiWarps = 16;
constexpr int kEpiThreads = kEpiWarps * 32;
constexpr int kFThreads = (2 + kEpiWarps) * 32;
constexpr float kL2e = 1.4426950408889634f;

struct FusedParams {
  int K, H, J;
  int tiles;        // (J / 128) * B * H
  float c;          // scale * log2(e)   (fwd)  |  scale  (bwd)
  int64_t g0;       // Philox chunk index of element (b=0,h=0,j=0,k=0) of this call
  const float* mask_bias;  // [B, K] or null (fwd)
};

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// bf16x8 pack of v[0..7]
__device__ __forceinline__ uint4 pack8(const float* v) {
  uint4 u;
  u.x = Chunk<__nv_bfloat16>::pack2(v[0], v[1]);
  u.y = Chunk<__nv_bfloat16>::pack2(v[2], v[3]);
  u.z = Chunk<__nv_bfloat16>::pack2(v[4], v[5]);
  u.w = Chunk<__nv_bfloat16>::pack2(v[6], v[7]);
  return u;
}

// shared-memory layout (bytes, from a 1024-aligned base)
//   [0, 16K)          Q / dC tile   [128 x 64] bf16, K-major SW128
//   [16K, 80K)        K / V  tile   [K x 64]   bf16, K-major SW128 (256-row boxes)
//   [80K, 80K+X)      fwd: 16 per-warp staging tiles of 8 KB (P and A, [32 x 64] each)
//                     bwd: P tile [128 x K] bf16 as K/64 boxes of [128 x 64] SW128; dS is
//                     staged in place of the P chunks it replaces
//   then: stats [2 tiles][4 slices][128 rows] float2, {fwd mask bias [512] float | bwd keep
//   bits [4][512] u32}, barriers, tmem slot
constexpr uint32_t kOpA = 0, kOpB = 16384, kOpX = 81920;

template <int K, bool kBwd>
constexpr uint32_t x_bytes() {
  return kBwd ? (uint32_t)kRows * K * 2 : (uint32_t)kEpiWarps * 8192;
}

template <int K, bool kBwd, bool kMask>
__device__ __forceinline__ void fused_body(const CUtensorMap& mapA, const CUtensorMap& mapB,
                                           const CUtensorMap& mapP, const CUtensorMap& mapO1,
                                           const CUtensorMap& mapO2, const FusedParams& prm,
                                           const PhiloxKey& pk, unsigned char* base) {
  constexpr int kHalves = K > 256 ? 2 : 1;
  constexpr int kNmma = K / kHalves;   // N per MMA instruction
  constexpr uint32_t kTcols = K;       // 256 or 512: a power of 2
  constexpr int W = K / 4;             // columns per epilogue warp (64 or 128)
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int mtiles = prm.J / kRows;

  float2* stats = reinterpret_cast<float2*>(base + kOpX + x_bytes<K, kBwd>());  // [2][4][128]
  float* mb = reinterpret_cast<float*>(stats + 2 * 4 * kRows);          // fwd: mask bias [512]
  uint32_t* kbs = reinterpret_cast<uint32_t*>(mb);                     // bwd: keep bits [4][512]
  uint64_t* op_full = reinterpret_cast<uint64_t*>(kbs + 4 * kEpiThreads);
  uint64_t* op_empty = op_full + 1;
  uint64_t* tm_full = op_full + 2;
  uint64_t* tm_empty = op_full + 3;
  uint64_t* p_full = op_full + 4;
  uint64_t* p_empty = op_full + 5;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(op_full + 6);

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&mapA);
    tc::prefetch_tmap(&mapB);
    tc::prefetch_tmap(&mapO1);
    if (kBwd) tc::prefetch_tmap(&mapP);
    if (!kBwd) tc::prefetch_tmap(&mapO2);
    mbar_init(op_full, 1);
    mbar_init(op_empty, 1);
    mbar_init(tm_full, 1);
    mbar_init(tm_empty, kEpiWarps);
    mbar_init(p_full, 1);
    mbar_init(p_empty, kEpiWarps);
    fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, kTcols);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int it = 0;
      for (int t = blockIdx.x; t < prm.tiles; t += gridDim.x, ++it) {
        const int bh = t / mtiles, m0 = (t - bh * mtiles) * kRows;
        const int b = bh / prm.H, h = bh - (bh / prm.H) * prm.H;
        mbar_wait(op_empty, (it & 1) ^ 1);
        mbar_arrive_expect_tx(op_full, (uint32_t)(kRows + K) * 128);
        if (!kBwd)
          tc::tma_load_4d(base + kOpA, &mapA, op_full, 0, m0, h, b);     // Q  [B,H,J,P]
        else
          tc::tma_load_4d(base + kOpA, &mapA, op_full, 0, h, m0, b);     // dC [B,J,H,P]
#pragma unroll
        for (int r = 0; r < K; r += 256)
          tc::tma_load_4d(base + kOpB + r * 128, &mapB, op_full, 0, r, h, b);  // K or V
        if (kBwd) {
          mbar_wait(p_empty, (it & 1) ^ 1);
          mbar_arrive_expect_tx(p_full, (uint32_t)kRows * K * 2);
#pragma unroll
          for (int c = 0; c < K; c += 64)
            tc::tma_load_4d(base + kOpX + c * 256, &mapP, p_full, c, m0, h, b);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = tc::instr_desc_bf16_f32(kRows, kNmma, false, false);
    const uint32_t a0 = smem_u32(base + kOpA), b0 = smem_u32(base + kOpB);
    int it = 0;
    for (int t = blockIdx.x; t < prm.tiles; t += gridDim.x, ++it) {
      mbar_wait(tm_empty, (it & 1) ^ 1);   // epilogue finished reading the accumulator
      mbar_wait(op_full, it & 1);
      tc::fence_after_sync();
      if (lane == 0) {
#pragma unroll
        for (int nh = 0; nh < kHalves; ++nh) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            tc::mma_bf16(tmem + nh * kNmma, tc::smem_desc(a0 + k * 32, 16, 1024),
                         tc::smem_desc(b0 + nh * kNmma * 128 + k * 32, 16, 1024), idesc, k != 0);
        }
        tc::mma_commit(op_empty);
        tc::mma_commit(tm_full);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int e = warp - 2;          // 0..15
    const int q = warp & 3;          // TMEM lane quarter
    const int slice = e >> 2;        // 0..3: columns [slice*W, (slice+1)*W)
    const int r = q * 32 + lane;     // row within the tile
    const int cb = slice * W;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16) + cb;
    unsigned char* stg = base + kOpX + e * 8192;   // fwd staging (P tile, A tile)
    int it = 0;
    for (int t = blockIdx.x; t < prm.tiles; t += gridDim.x, ++it) {
      const int bh = t / mtiles, m0 = (t - bh * mtiles) * kRows;
      const int b = bh / prm.H, h = bh - (bh / prm.H) * prm.H;
      const int64_t grow = prm.g0 + ((int64_t)bh * prm.J + m0 + r) * (K / 8) + cb / 8;
      float2* st = stats + (it & 1) * 4 * kRows;
      if (kMask) {   // additive mask bias of this b, pre-multiplied by log2(e)
        named_bar(5, kEpiThreads);   // previous tile's readers are done
        for (int k = threadIdx.x - 64; k < K; k += kEpiThreads)
          mb[k] = prm.mask_bias[(int64_t)b * K + k] * kL2e;
        named_bar(5, kEpiThreads);
      }
      mbar_wait(tm_full, it & 1);
      tc::fence_after_sync();
      if (!kBwd) {
        const float c = prm.c;
        // pass 1: row max of y = scale*log2e*S (+ mask*log2e) over this slice
        float m = -INFINITY;
#pragma unroll 1
        for (int c0 = 0; c0 < W; c0 += 32) {
          float v[32];
          tc::tmem_ld32(trow + c0, v);
#pragma unroll
          for (int i = 0; i < 32; ++i)
            m = fmaxf(m, kMask ? fmaf(v[i], c, mb[cb + c0 + i]) : v[i] * c);
        }
        st[slice * kRows + r].x = m;
        named_bar(1 + q, 128);
        float M = st[r].x;
#pragma unroll
        for (int s = 1; s < 4; ++s) M = fmaxf(M, st[s * kRows + r].x);
        // pass 2: e = 2^(y - M) (one MUFU per element) back into TMEM, row sum
        float l = 0.f;
#pragma unroll 1
        for (int c0 = 0; c0 < W; c0 += 32) {
          float v[32];
          tc::tmem_ld32(trow + c0, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            v[i] = tc::ex2(kMask ? fmaf(v[i], c, mb[cb + c0 + i] - M) : fmaf(v[i], c, -M));
            l += v[i];
          }
          tc::tmem_st32(trow + c0, v);
        }
        tc::tmem_wait_st();
        st[slice * kRows + r].y = l;
        named_bar(1 + q, 128);
        float L = 0.f;
#pragma unroll
        for (int s = 0; s < 4; ++s) L += st[s * kRows + r].y;
        const float inv = __fdividef(1.f, L);
        // pass 3: P = e / L and A = dropout(P), 64 columns per staging round
#pragma unroll 1
        for (int c0 = 0; c0 < W; c0 += 64) {
          if (lane == 0) tc::bulk_wait_read<0>();   // staging tile free again
          __syncwarp();
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            float v[32];
            tc::tmem_ld32(trow + c0 + 32 * half, v);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              float* x = v + 8 * j;
#pragma unroll
              for (int u = 0; u < 8; ++u) x[u] *= inv;
              *reinterpret_cast<uint4*>(stg + tc::sw128(lane, half * 4 + j)) = pack8(x);
              dropout8(x, (uint64_t)(grow + (c0 + 32 * half) / 8 + j), pk);
              *reinterpret_cast<uint4*>(stg + 4096 + tc::sw128(lane, half * 4 + j)) = pack8(x);
            }
          }
          if (c0 + 64 >= W) {   // last TMEM read of this tile by this warp
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) mbar_arrive(tm_empty);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tc::tma_store_4d(&mapO1, stg, cb + c0, m0 + q * 32, h, b);
            tc::tma_store_4d(&mapO2, stg + 4096, cb + c0, m0 + q * 32, h, b);
            tc::bulk_commit();
          }
        }
      } else {
        // pass 1: dot = sum_k dropout(dA)_k * P_k over this slice
        mbar_wait(p_full, it & 1);
        unsigned char* sP = base + kOpX;
        uint32_t* kbits = kbs + (threadIdx.x - 64);   // [W/32] words, stride 512 threads
        float dot = 0.f;
#pragma unroll 1
        for (int c0 = 0; c0 < W; c0 += 32) {
          float v[32];
          tc::tmem_ld32(trow + c0, v);
          uint32_t word = 0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int cc = cb + c0 + 8 * j;
            float mk[8], p[8];
            keep_mul8((uint64_t)(grow + (c0 + 8 * j) / 8), pk, mk);
#pragma unroll
            for (int u = 0; u < 8; ++u) word |= (mk[u] != 0.f ? 1u : 0u) << (8 * j + u);
            Chunk<__nv_bfloat16>::unpack(
                *reinterpret_cast<const uint4*>(sP + (cc >> 6) * 16384 + tc::sw128(r, (cc & 63) >> 3)), p);
#pragma unroll
            for (int u = 0; u < 8; ++u) dot = fmaf(v[8 * j + u] * mk[u], p[u], dot);
          }
          kbits[(c0 / 32) * kEpiThreads] = word;
        }
        st[slice * kRows + r].x = dot;
        named_bar(1 + q, 128);
        float D = 0.f;
#pragma unroll
        for (int s = 0; s < 4; ++s) D += st[s * kRows + r].x;
        const float sc = pk.scale, scale = prm.c;
        // pass 2: dS = scale * P * (dP - D), written over the P chunk it came from; each
        // 64-column group of this warp is a contiguous [32 x 64] sub-tile of a P box
#pragma unroll 1
        for (int c0 = 0; c0 < W; c0 += 64) {
          const int cg = cb + c0;                       // multiple of 64
          unsigned char* sub = sP + (cg >> 6) * 16384 + q * 4096;
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            float v[32];
            tc::tmem_ld32(trow + c0 + 32 * half, v);
            const uint32_t word = kbits[((c0 + 32 * half) / 32) * kEpiThreads];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              float p[8], o[8];
              uint4* loc = reinterpret_cast<uint4*>(sub + tc::sw128(lane, half * 4 + j));
              Chunk<__nv_bfloat16>::unpack(*loc, p);
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const float dp = ((word >> (8 * j + u)) & 1u) ? v[8 * j + u] * sc : 0.f;
                o[u] = scale * p[u] * (dp - D);
              }
              *loc = pack8(o);
            }
          }
          if (c0 + 64 >= W) {   // last TMEM read of this tile by this warp
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) mbar_arrive(tm_empty);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tc::tma_store_4d(&mapO1, sub, cg, m0 + q * 32, h, b);
            tc::bulk_commit();
          }
        }
        // the next tile's P may overwrite this warp's sub-tiles once the stores read them
        if (lane == 0) {
          tc::bulk_wait_read<0>();
          mbar_arrive(p_empty);
        }
        __syncwarp();
      }
    }
    if (lane == 0) tc::bulk_wait<0>();
    __syncwarp();
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, kTcols);
}

template <int K, bool kMask>
__global__ void __launch_bounds__(kFThreads, 1) attn_qk_bsb_kernel(
    const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapK,
    const __grid_constant__ CUtensorMap mapP, const __grid_constant__ CUtensorMap mapA,
    FusedParams prm, PhiloxKey pk) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  fused_body<K, false, kMask>(mapQ, mapK, mapQ, mapP, mapA, prm, pk, tc::align1024(smem_raw));
}

template <int K>
__global__ void __launch_bounds__(kFThreads, 1) attn_da_bsbb_kernel(
    const __grid_constant__ CUtensorMap mapdC, const __grid_constant__ CUtensorMap mapV,
    const __grid_constant__ CUtensorMap mapP, const __grid_constant__ CUtensorMap mapdS,
    FusedParams prm, PhiloxKey pk) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  fused_body<K, true, false>(mapdC, mapV, mapP, mapdS, mapdS, prm, pk, tc::align1024(smem_raw));
}

template <int K, bool kBwd>
constexpr size_t fused_smem() {
  return 1024 + kOpX + x_bytes<K, kBwd>() + 2 * 4 * kRows * sizeof(float2) +
         4 * kEpiThreads * sizeof(uint32_t) + 8 * sizeof(uint64_t);  // mb | kbs union
}
static_assert(fused_smem<512, true>() <= 227 * 1024, "bwd smem");
static_assert(fused_smem<512, false>() <= 227 * 1024, "fwd smem");

bool map4(CUtensorMap* m, const void* ptr, const uint64_t d[4], const uint64_t s[3],
          const uint32_t box[4]) {
  cuuint64_t gdim[4] = {d[0], d[1], d[2], d[3]};
  cuuint64_t gstr[3] = {s[0] * 2, s[1] * 2, s[2] * 2};
  cuuint32_t bdim[4] = {box[0], box[1], box[2], box[3]};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return tmap_encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), gdim,
                           gstr, bdim, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// [B][H][rows][cols] with box {64, box_rows}
bool map_bhrc(CUtensorMap* m, const void* p, int B, int H, int rows, int cols, int box_rows) {
  const uint64_t d[4] = {(uint64_t)cols, (uint64_t)rows, (uint64_t)H, (uint64_t)B};
  const uint64_t s[3] = {(uint64_t)cols, (uint64_t)rows * cols, (uint64_t)H * rows * cols};
  const uint32_t box[4] = {64, (uint32_t)box_rows, 1, 1};
  return map4(m, p, d, s, box);
}

// [B][rows][H][cols] (cols = P) with box {64, 1, box_rows, 1}
bool map_brhc(CUtensorMap* m, const void* p, int B, int H, int rows, int cols, int box_rows) {
  const uint64_t d[4] = {(uint64_t)cols, (uint64_t)H, (uint64_t)rows, (uint64_t)B};
  const uint64_t s[3] = {(uint64_t)cols, (uint64_t)H * cols, (uint64_t)rows * H * cols};
  const uint32_t box[4] = {64, 1, (uint32_t)box_rows, 1};
  return map4(m, p, d, s, box);
}

int persistent_grid(int tiles) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms <= 0) sms = 148;
  return tiles < sms ? tiles : sms;
}

template <typename Kern>
cudaError_t launch_persistent(Kern kern, size_t smem, int tiles, const CUtensorMap& a,
                              const CUtensorMap& b, const CUtensorMap& c, const CUtensorMap& d,
                              const FusedParams& prm, const PhiloxKey& pk, cudaStream_t st) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<persistent_grid(tiles), kFThreads, smem, st>>>(a, b, c, d, prm, pk);
  return cudaGetLastError();
}

}  // namespace

// K = J in {256, 512}: the K operand is loaded as whole 256-row boxes and each of the 4
// column slices of a row spans a multiple of 64 columns (one staging tile)
bool attn_fused_supported(int J, int P) { return P == 64 && (J == 256 || J == 512); }

cudaError_t launch_attn_qk_bsb(int B, int H, int J, int P, float scale, const void* Q,
                               const void* Kt, const float* mask_bias, const PhiloxKey& pk,
                               int64_t batch_offset, void* Pout, void* Aout, cudaStream_t st) {
  const int K = J;
  CUtensorMap mq, mk, mp, ma;
  bool ok = map_bhrc(&mq, Q, B, H, J, P, kRows) && map_bhrc(&mk, Kt, B, H, K, P, 256) &&
            map_bhrc(&mp, Pout, B, H, J, K, 32) && map_bhrc(&ma, Aout, B, H, J, K, 32);
  if (!ok) return cudaErrorInvalidValue;
  const int tiles = (J / kRows) * B * H;
  FusedParams prm{K, H, J, tiles, scale * kL2e, batch_offset * (int64_t)H * J * (K / 8),
                  mask_bias};
  if (K == 512)
    return mask_bias ? launch_persistent(attn_qk_bsb_kernel<512, true>, fused_smem<512, false>(),
                                         tiles, mq, mk, mp, ma, prm, pk, st)
                     : launch_persistent(attn_qk_bsb_kernel<512, false>, fused_smem<512, false>(),
                                         tiles, mq, mk, mp, ma, prm, pk, st);
  return mask_bias ? launch_persistent(attn_qk_bsb_kernel<256, true>, fused_smem<256, false>(),
                                       tiles, mq, mk, mp, ma, prm, pk, st)
                   : launch_persistent(attn_qk_bsb_kernel<256, false>, fused_smem<256, false>(),
                                       tiles, mq, mk, mp, ma, prm, pk, st);
}

cudaError_t launch_attn_da_bsbb(int B, int H, int J, int P, float scale, const void* dC,
                                const void* V, const void* Pin, const PhiloxKey& pk,
                                int64_t batch_offset, void* dS, cudaStream_t st) {
  const int K = J;
  CUtensorMap mc, mv, mp, ms;
  bool ok = map_brhc(&mc, dC, B, H, J, P, kRows) && map_bhrc(&mv, V, B, H, K, P, 256) &&
            map_bhrc(&mp, Pin, B, H, J, K, kRows) && map_bhrc(&ms, dS, B, H, J, K, 32);
  if (!ok) return cudaErrorInvalidValue;
  const int tiles = (J / kRows) * B * H;
  FusedParams prm{K, H, J, tiles, scale, batch_offset * (int64_t)H * J * (K / 8), nullptr};
  if (K == 512)
    return launch_persistent(attn_da_bsbb_kernel<512>, fused_smem<512, true>(), tiles, mc, mv,
                             mp, ms, prm, pk, st);
  return launch_persistent(attn_da_bsbb_kernel<256>, fused_smem<256, true>(), tiles, mc, mv, mp,
                           ms, prm, pk, st);
}

}  // namespace enc

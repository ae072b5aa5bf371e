// Fused score kernels for short sequences, J = K = 128, P = 64 (BERT-base, BASELINE config
// Bb): the J = 512 kernels of attn_fused.cu fill all 512 TMEM columns with one 128-row tile;
// at K = 128 a whole (b, h) score matrix is one 128 x 128 MMA tile, so four of them fit in
// TMEM at once and the kernel pipelines (b, h) pairs through TMEM slots.
//
//  attn_qk_bsb_short  S = Q K^T (Table A.1 :551) -> BSB (`sm`, :552): writes P and the keep
//                     words (ENC_KEEP_BITS); A = dropout(P) is applied on load by the
//                     per-(b,h) A.V / A^T.dC contractions (attn_bh.cu), so it is not stored.
//                     Saves the S write + read of the unfused pair (2 x 37.7 MB at Bb).
//  attn_da_bsbb_short dA = dC V^T (:588) -> BSB-bwd (`bs`, :590) with the saved P and keep
//                     words: writes dS.  Saves the dA write + read (2 x 37.7 MB at Bb).
//
// Persistent CTAs, one per SM.  Warp 0 lane 0 is the TMA producer and tcgen05.mma issuer
// (M = 128, N = 128, K = 16 x 4); 4 x kSlots epilogue warps (warps 4..): warp w serves TMEM
// slot (w - 4) / 4 (columns slot * 128 ..) and lane quarter w % 4.  Tile i of a CTA uses
// slot i % kSlots, so the MMA of one (b, h) pair overlaps the epilogues of the others.
// Epilogue thread = one score row (128 keys): the softmax statistics are thread-local (no
// cross-warp reduction): pass 1 per 32-key chunk: y = scale*log2e*S (+ mask), chunk max
// m_c, e = 2^(y - m_c) back into TMEM, chunk sum l_c; pass 2: P = e 2^(m_c - M) / L.
// Backward pass 1: dot = sum_k keep dA P (P from shared memory), pass 2: dS = scale P
// (keep s dA - s dot) written over P in shared memory and stored by TMA.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "kernels.h"
#include "tc_gemm.cuh"

namespace enc {
namespace {

constexpr int kS = 128;                     // J = K
constexpr float kL2e = 1.4426950408889634f;

struct ShortParams {
  int H, tiles;            // tiles = B * H (one (b, h) pair each)
  float c;                 // fwd: scale * log2(e); bwd: scale
  int64_t g0;              // Philox chunk index of element (b=0,h=0,j=0,k=0) of this call
  const float* mask_bias;  // [B, K] or null (fwd)
  uint32_t* keep_bits;     // [B, H, J, K/32] or null (fwd: written, or read if keep_pre;
                           // bwd: read, or the flags regenerated from Philox if null)
  int causal, write_a, keep_pre;
};

__device__ __forceinline__ uint4 pack8(const float* v) {
  uint4 u;
  u.x = Chunk<__nv_bfloat16>::pack2(v[0], v[1]);
  u.y = Chunk<__nv_bfloat16>::pack2(v[2], v[3]);
  u.z = Chunk<__nv_bfloat16>::pack2(v[4], v[5]);
  u.w = Chunk<__nv_bfloat16>::pack2(v[6], v[7]);
  return u;
}
__device__ __forceinline__ uint32_t sw64(int r, int c) {
  return (uint32_t)(r * 64 + ((c ^ ((r >> 1) & 3)) << 4));
}
// keep_flags: common.cuh
__device__ __forceinline__ constexpr int flag_bit(int j, int u) {
  return ((u & 1) ? 31 : 15) - (u >> 1) - 4 * j;
}
// the 4 keep words of one 128-key row whose first Philox chunk is `grow`
__device__ __forceinline__ void row_flags(uint32_t kf[4], int64_t grow, const PhiloxKey& pk,
                                          uint32_t C2, uint32_t X) {
  if (pk.T == 0) {   // p = 0: everything kept, no Philox stream
    kf[0] = kf[1] = kf[2] = kf[3] = 0xFFFFFFFFu;
    return;
  }
#pragma unroll
  for (int w4 = 0; w4 < 4; ++w4) {
    uint32_t f = 0;
#pragma unroll 2
    for (int j = 0; j < 4; ++j) f |= keep_flags((uint64_t)(grow + 4 * w4 + j), pk, C2, X, 4 * j);
    kf[w4] = f;
  }
}

// ------------------------------------------------------------------ forward
constexpr int kFSlots = 3;
constexpr int kFThreads = 32 * (4 + 4 * kFSlots);
constexpr uint32_t kOpBytes = kS * 64 * 2;   // one 128 x 64 bf16 operand tile (16 KB)
constexpr uint32_t kStg = 32 * 64;           // [32 rows x 64 B] staging buffer
constexpr size_t kFSmem = 1024 + (size_t)kFSlots * 2 * kOpBytes + 4 * kFSlots * 2 * kStg + 256;

template <bool kMask, bool kCausal>
__global__ void __launch_bounds__(kFThreads, 1) attn_qk_bsb_short_kernel(
    const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapK,
    const __grid_constant__ CUtensorMap mapP, const __grid_constant__ CUtensorMap mapA,
    ShortParams prm, PhiloxKey pk) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = tc::align1024(smem_raw);
  unsigned char* stg_all = base + kFSlots * 2 * kOpBytes;
  uint64_t* op_full = reinterpret_cast<uint64_t*>(stg_all + 4 * kFSlots * 2 * kStg);
  uint64_t* op_empty = op_full + kFSlots;
  uint64_t* tm_full = op_empty + kFSlots;
  uint64_t* tm_empty = tm_full + kFSlots;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tm_empty + kFSlots);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = prm.H;

  if (threadIdx.x == 0) {
    tc::prefetch_tmap(&mapQ);
    tc::prefetch_tmap(&mapK);
    tc::prefetch_tmap(&mapP);
    if (prm.write_a) tc::prefetch_tmap(&mapA);
    for (int s = 0; s < kFSlots; ++s) {
      mbar_init(&op_full[s], 1);
      mbar_init(&op_empty[s], 1);
      mbar_init(&tm_full[s], 1);
      mbar_init(&tm_empty[s], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();   // operands are the stream predecessor's outputs

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------- producer + MMA
      auto load = [&](int t, int s) {
        const int b = t / H, h = t - b * H;
        unsigned char* a = base + s * 2 * kOpBytes;
        mbar_arrive_expect_tx(&op_full[s], 2 * kOpBytes);
        tc::tma_load_4d(a, &mapQ, &op_full[s], 0, h, 0, b);             // Q rows 0..127
        tc::tma_load_4d(a + kOpBytes, &mapK, &op_full[s], 0, h, 0, b);  // K rows 0..127
      };
      int i = 0;
      for (int t = blockIdx.x; t < prm.tiles && i < kFSlots; t += gridDim.x, ++i) load(t, i);
      constexpr uint32_t idesc = tc::instr_desc_bf16_f32(kS, kS, false, false);
      i = 0;
      for (int t = blockIdx.x; t < prm.tiles; t += gridDim.x, ++i) {
        const int s = i % kFSlots;
        const uint32_t ph = (uint32_t)(i / kFSlots) & 1u;
        mbar_wait(&tm_empty[s], ph ^ 1u);
        mbar_wait(&op_full[s], ph);
        tc::fence_after_sync();
        const uint64_t ad = tc::smem_desc(smem_u32(base + s * 2 * kOpBytes), 16, 1024);
        const uint64_t bd = tc::desc_adv(ad, kOpBytes);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc::mma_bf16(tmem + s * kS, tc::desc_adv(ad, k * 32), tc::desc_adv(bd, k * 32), idesc,
                       k != 0);
        tc::mma_commit(&tm_full[s]);
        tc::mma_commit(&op_empty[s]);
        const int tn = t + kFSlots * (int)gridDim.x;
        if (tn < prm.tiles) {   // the slot's operands are free once these MMAs finished
          mbar_wait(&op_empty[s], ph);
          load(tn, s);
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------- epilogue
    const int ew = warp - 4, s = ew >> 2, q = warp & 3;
    const int r = q * 32 + lane;              // query row of this thread
    unsigned char* stg = stg_all + ew * 2 * kStg;
    const bool hiT = pk.T >= 0x8000u;
    const uint32_t C2 = (hiT ? 0x10000u - pk.T : 0x8000u - pk.T) * 0x10001u;
    const uint32_t X = hiT ? 0u : 0xFFFFFFFFu;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16) + s * kS;
    const float c = prm.c;
    uint32_t sc = 0;   // staging buffer parity
    int i = s;
    for (int t = blockIdx.x + s * (int)gridDim.x; t < prm.tiles;
         t += kFSlots * (int)gridDim.x, i += kFSlots) {
      const int b = t / H, h = t - b * H;
      const uint32_t ph = (uint32_t)(i / kFSlots) & 1u;
      // keep words of this row (independent of the MMA)
      const int64_t rowi = (int64_t)t * kS + r;
      uint32_t kf[4];
      if (prm.keep_pre) {
        const uint4 kw = __ldcs(reinterpret_cast<const uint4*>(prm.keep_bits + rowi * 4));
        kf[0] = kw.x, kf[1] = kw.y, kf[2] = kw.z, kf[3] = kw.w;
      } else if (!prm.keep_bits && !prm.write_a) {
        // neither A nor keep words stored (the layer's path: A.V generates the mask on load,
        // DESIGN.md R28): the flags are unused
        kf[0] = kf[1] = kf[2] = kf[3] = 0xFFFFFFFFu;
      } else {
        row_flags(kf, prm.g0 + rowi * (kS / 8), pk, C2, X);
        if (prm.keep_bits)
          __stcs(reinterpret_cast<uint4*>(prm.keep_bits + rowi * 4),
                 make_uint4(kf[0], kf[1], kf[2], kf[3]));
      }
      mbar_wait_sleep(&tm_full[s], ph, 20000u);
      tc::fence_after_sync();
      // pass 1: chunk max / exp2 back into TMEM / chunk sum
      float mc[4], lc[4], v[32];
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        tc::tmem_ld32(trow + ch * 32, v);
        if (kMask) {
          const float4* mb4 = reinterpret_cast<const float4*>(prm.mask_bias + (int64_t)b * kS + ch * 32);
#pragma unroll
          for (int k4 = 0; k4 < 8; ++k4) {
            const float4 mm = __ldg(mb4 + k4);
            v[4 * k4 + 0] = fmaf(v[4 * k4 + 0], c, mm.x * kL2e);
            v[4 * k4 + 1] = fmaf(v[4 * k4 + 1], c, mm.y * kL2e);
            v[4 * k4 + 2] = fmaf(v[4 * k4 + 2], c, mm.z * kL2e);
            v[4 * k4 + 3] = fmaf(v[4 * k4 + 3], c, mm.w * kL2e);
          }
        }
        if (kCausal) {   // keys after the query row are masked out
#pragma unroll
          for (int k = 0; k < 32; ++k)
            if (ch * 32 + k > r) v[k] = -INFINITY;
        }
        float m = tree_max<32>(v);
        if (!kMask) m *= c;   // c > 0: scale after the max
        // a fully masked chunk has m = -inf: exponentiate against 0 instead
        const float mz = m == -INFINITY ? 0.f : m;
#pragma unroll
        for (int k = 0; k < 32; ++k) v[k] = tc::ex2(kMask ? v[k] - mz : fmaf(v[k], c, -mz));
        mc[ch] = m;
        lc[ch] = tree_sum<32>(v);
        tc::tmem_st32(trow + ch * 32, v);
      }
      tc::tmem_wait_st();
      float M = fmaxf(fmaxf(mc[0], mc[1]), fmaxf(mc[2], mc[3]));
      const float Mr = M == -INFINITY ? 0.f : M;
      float L = 0.f;
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) L += lc[ch] * tc::ex2((mc[ch] == -INFINITY ? 0.f : mc[ch]) - Mr);
      const float invL = __fdividef(1.f, L);
      // pass 2: P = e 2^(m_c - M) / L, staged per 32 columns and stored by TMA
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        tc::tmem_ld32(trow + ch * 32, v);
        if (ch == 3) {   // accumulator drained
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tm_empty[s]);
        }
        const float fp = tc::ex2((mc[ch] == -INFINITY ? 0.f : mc[ch]) - Mr) * invL;
        const float fa = fp * pk.scale;
        // P alone: the two staging buffers alternate; P and A: one buffer each per round
        unsigned char* sb = stg + (prm.write_a ? 0u : (sc & 1) * kStg);
        if (lane == 0) {   // the buffer's previous store has read it
          if (prm.write_a) tc::bulk_wait_read<0>();
          else tc::bulk_wait_read<1>();
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float x[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) x[u] = v[8 * j + u] * fp;
          *reinterpret_cast<uint4*>(sb + sw64(lane, j)) = pack8(x);
          if (prm.write_a) {
#pragma unroll
            for (int u = 0; u < 8; ++u)
              x[u] = ((kf[ch] >> flag_bit(j, u)) & 1u) ? v[8 * j + u] * fa : 0.f;
            *reinterpret_cast<uint4*>(sb + kStg + sw64(lane, j)) = pack8(x);
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tc::tma_store_4d(&mapP, sb, ch * 32, q * 32, h, b);
          if (prm.write_a) tc::tma_store_4d(&mapA, sb + kStg, ch * 32, q * 32, h, b);
          tc::bulk_commit();
        }
        ++sc;
      }
    }
    if (lane == 0) tc::bulk_wait<0>();
    __syncwarp();
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// ------------------------------------------------------------------ backward
// Three epilogue groups (TMEM slots), with the loads decoupled from them: a 2-stage ring of
// dC / V operand tiles (free once the MMA read them) and a 5-deep ring of P tiles (free once
// the dS written over them has been read out by the TMA store), each filled by its own
// producer thread, so up to two tiles' P loads are in flight beside the three epilogues.
constexpr int kBSlots = 3;                   // TMEM slots = epilogue groups
constexpr int kBOps = 2;                     // dC / V operand stages
constexpr int kBPs = 5;                      // P / dS tile buffers
constexpr int kBThreads = 32 * (4 + 4 * kBSlots);
constexpr uint32_t kPBytes = kS * kS * 2;    // P / dS tile (32 KB): [4 quarters][2 halves][32 x 128 B]
constexpr uint32_t kBOpOff = kBPs * kPBytes;
constexpr uint32_t kBBarOff = kBOpOff + kBOps * 2 * kOpBytes;
constexpr size_t kBSmem = 1024 + kBBarOff + 8 * (2 * kBOps + 2 * kBPs + 2 * kBSlots) + 16;
static_assert(kBSmem <= 232448, "smem");

__global__ void __launch_bounds__(kBThreads, 1) attn_da_bsbb_short_kernel(
    const __grid_constant__ CUtensorMap mapdC, const __grid_constant__ CUtensorMap mapV,
    const __grid_constant__ CUtensorMap mapP, const __grid_constant__ CUtensorMap mapdS,
    ShortParams prm, PhiloxKey pk) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = tc::align1024(smem_raw);
  uint64_t* op_full = reinterpret_cast<uint64_t*>(base + kBBarOff);
  uint64_t* op_empty = op_full + kBOps;       // MMA read the operands
  uint64_t* p_full = op_empty + kBOps;
  uint64_t* p_free = p_full + kBPs;           // the 4 warps' dS stores have read the buffer
  uint64_t* tm_full = p_free + kBPs;
  uint64_t* tm_empty = tm_full + kBSlots;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tm_empty + kBSlots);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = prm.H;
  const int G = (int)gridDim.x;
  const int ntiles = prm.tiles > (int)blockIdx.x ? (prm.tiles - (int)blockIdx.x + G - 1) / G : 0;

  if (threadIdx.x == 0) {
    tc::prefetch_tmap(&mapdC);
    tc::prefetch_tmap(&mapV);
    tc::prefetch_tmap(&mapP);
    tc::prefetch_tmap(&mapdS);
    for (int s = 0; s < kBOps; ++s) {
      mbar_init(&op_full[s], 1);
      mbar_init(&op_empty[s], 1);
    }
    for (int s = 0; s < kBPs; ++s) {
      mbar_init(&p_full[s], 1);
      mbar_init(&p_free[s], 4);
    }
    for (int s = 0; s < kBSlots; ++s) {
      mbar_init(&tm_full[s], 1);
      mbar_init(&tm_empty[s], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();   // operands are the stream predecessor's outputs

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------- operands + MMA
      auto load = [&](int i) {
        const int t = (int)blockIdx.x + i * G, s = i % kBOps;
        const int b = t / H, h = t - b * H;
        unsigned char* a = base + kBOpOff + s * 2 * kOpBytes;
        mbar_arrive_expect_tx(&op_full[s], 2 * kOpBytes);
        tc::tma_load_4d(a, &mapdC, &op_full[s], 0, h, 0, b);             // dC rows 0..127
        tc::tma_load_4d(a + kOpBytes, &mapV, &op_full[s], 0, h, 0, b);   // V rows 0..127
      };
      for (int i = 0; i < ntiles && i < kBOps; ++i) load(i);
      constexpr uint32_t idesc = tc::instr_desc_bf16_f32(kS, kS, false, false);
      for (int i = 0; i < ntiles; ++i) {
        const int so = i % kBOps, st = i % kBSlots;
        mbar_wait(&tm_empty[st], ((uint32_t)(i / kBSlots) & 1u) ^ 1u);
        mbar_wait(&op_full[so], (uint32_t)(i / kBOps) & 1u);
        tc::fence_after_sync();
        const uint64_t ad = tc::smem_desc(smem_u32(base + kBOpOff + so * 2 * kOpBytes), 16, 1024);
        const uint64_t bd = tc::desc_adv(ad, kOpBytes);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc::mma_bf16(tmem + st * kS, tc::desc_adv(ad, k * 32), tc::desc_adv(bd, k * 32), idesc,
                       k != 0);
        tc::mma_commit(&tm_full[st]);
        tc::mma_commit(&op_empty[so]);
        if (i + kBOps < ntiles) {   // the stage is free once these MMAs have read it
          mbar_wait(&op_empty[so], (uint32_t)(i / kBOps) & 1u);
          load(i + kBOps);
        }
      }
    }
  } else if (warp == 2) {
    if (lane == 0) {
      // ---------------------------------------------------------- P tiles
      for (int i = 0; i < ntiles; ++i) {
        const int t = (int)blockIdx.x + i * G, sp = i % kBPs;
        const int b = t / H, h = t - b * H;
        mbar_wait(&p_free[sp], ((uint32_t)(i / kBPs) & 1u) ^ 1u);
        mbar_arrive_expect_tx(&p_full[sp], kPBytes);
        unsigned char* pt = base + sp * kPBytes;
#pragma unroll
        for (int qq = 0; qq < 4; ++qq)
#pragma unroll
          for (int hf = 0; hf < 2; ++hf)
            tc::tma_load_4d(pt + (qq * 2 + hf) * 4096, &mapP, &p_full[sp], hf * 64, qq * 32, h, b);
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4, s = ew >> 2, q = warp & 3;
    const int r = q * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16) + s * kS;
    const float ss = prm.c * pk.scale;   // scale * dropout scale
    const bool hiT = pk.T >= 0x8000u;
    const uint32_t C2 = (hiT ? 0x10000u - pk.T : 0x8000u - pk.T) * 0x10001u;
    const uint32_t X = hiT ? 0u : 0xFFFFFFFFu;
    int pending = -1;   // P buffer whose dS store this warp has not yet released
    for (int i = s; i < ntiles; i += kBSlots) {
      const int t = (int)blockIdx.x + i * G, sp = i % kBPs;
      const int b = t / H, h = t - b * H;
      const int64_t rowi = (int64_t)t * kS + r;
      uint32_t kf[4];
      if (prm.keep_bits) {
        const uint4 kw = __ldcs(reinterpret_cast<const uint4*>(prm.keep_bits + rowi * 4));
        kf[0] = kw.x, kf[1] = kw.y, kf[2] = kw.z, kf[3] = kw.w;
      } else {
        row_flags(kf, prm.g0 + rowi * (kS / 8), pk, C2, X);
      }
      if (pending >= 0 && lane == 0) {   // release the previous tile's buffer (deferred)
        tc::bulk_wait_read<0>();
        mbar_arrive(&p_free[pending]);
      }
      mbar_wait_sleep(&tm_full[s], (uint32_t)(i / kBSlots) & 1u, 20000u);
      mbar_wait(&p_full[sp], (uint32_t)(i / kBPs) & 1u);
      tc::fence_after_sync();
      unsigned char* pt = base + sp * kPBytes + q * 2 * 4096;
      // pass 1: dot = sum_k keep_k dA_k P_k (four partial sums)
      float v[32], dacc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        tc::tmem_ld32(trow + ch * 32, v);
        const unsigned char* half = pt + (ch >> 1) * 4096;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float p[8];
          Chunk<__nv_bfloat16>::unpack(
              *reinterpret_cast<const uint4*>(half + tc::sw128(lane, (ch & 1) * 4 + j)), p);
#pragma unroll
          for (int u = 0; u < 8; ++u)
            dacc[u & 3] = fmaf(((kf[ch] >> flag_bit(j, u)) & 1u) ? v[8 * j + u] : 0.f, p[u],
                               dacc[u & 3]);
        }
      }
      const float dot = (dacc[0] + dacc[1]) + (dacc[2] + dacc[3]);
      const float nDs = -dot * ss;
      // pass 2: dS = P (keep ? scale s dA : 0) - scale s dot P, in place of P
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        tc::tmem_ld32(trow + ch * 32, v);
        if (ch == 3) {
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tm_empty[s]);
        }
        unsigned char* half = pt + (ch >> 1) * 4096;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint4* loc = reinterpret_cast<uint4*>(half + tc::sw128(lane, (ch & 1) * 4 + j));
          float p[8];
          Chunk<__nv_bfloat16>::unpack(*loc, p);
#pragma unroll
          for (int u = 0; u < 8; ++u)
            p[u] *= ((kf[ch] >> flag_bit(j, u)) & 1u) ? fmaf(v[8 * j + u], ss, nDs) : nDs;
          *loc = pack8(p);
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tc::tma_store_4d(&mapdS, pt, 0, q * 32, h, b);
        tc::tma_store_4d(&mapdS, pt + 4096, 64, q * 32, h, b);
        tc::bulk_commit();
      }
      pending = sp;
      __syncwarp();
    }
    if (lane == 0) tc::bulk_wait<0>();
    __syncwarp();
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

bool map_bhrc_s(CUtensorMap* m, const void* p, int B, int H, int rows, int cols, int box_cols,
                int box_rows, CUtensorMapSwizzle sw) {
  cuuint64_t gdim[4] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)H, (cuuint64_t)B};
  cuuint64_t gstr[3] = {(cuuint64_t)cols * 2, (cuuint64_t)rows * cols * 2,
                        (cuuint64_t)H * rows * cols * 2};
  cuuint32_t bdim[4] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return tmap_encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(p), gdim,
                           gstr, bdim, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int sms_of_device() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

template <typename Kern, typename... Args>
cudaError_t launch_short(Kern kern, int tiles, size_t smem, int threads, cudaStream_t st,
                         bool high_prio, Args... args) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int sms = sms_of_device();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tiles < sms ? tiles : sms);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (high_prio) {   // placed ahead of a kernel made ready on another stream (layer dV)
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    at[na].id = cudaLaunchAttributePriority;
    at[na++].val.priority = greatest;
  }
  if (pdl_enabled(PDL_ATTN_FUSED)) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na++].val.programmaticStreamSerializationAllowed = 1;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

}  // namespace

bool attn_short_supported(int J, int P) { return J == kS && P == 64; }

cudaError_t launch_attn_qk_bsb_short(int B, int H, int J, int P, float scale, const void* Q,
                                     int64_t ldq, const void* Kt, int64_t ldk,
                                     const float* mask_bias, const PhiloxKey& pk,
                                     int64_t batch_offset, void* Pout, void* Aout,
                                     uint32_t* keep_bits, cudaStream_t st, int causal,
                                     int keep_pre) {
  if (!attn_short_supported(J, P) || (keep_pre && !keep_bits)) return cudaErrorInvalidValue;
  CUtensorMap mq, mk, mp, ma;
  bool ok = map_pop(&mq, Q, B, H, J, P, ldq, kS) && map_pop(&mk, Kt, B, H, J, P, ldk, kS) &&
            map_bhrc_s(&mp, Pout, B, H, J, J, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B) &&
            map_bhrc_s(&ma, Aout ? Aout : Pout, B, H, J, J, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
  if (!ok) return cudaErrorInvalidValue;
  const int tiles = B * H;
  ShortParams prm{H,         tiles,     scale * kL2e, batch_offset * (int64_t)H * J * (J / 8),
                  mask_bias, keep_bits, causal,       Aout != nullptr,
                  keep_pre ? 1 : 0};
  if (causal)
    return mask_bias ? launch_short(attn_qk_bsb_short_kernel<true, true>, tiles, kFSmem, kFThreads,
                                    st, false, mq, mk, mp, ma, prm, pk)
                     : launch_short(attn_qk_bsb_short_kernel<false, true>, tiles, kFSmem,
                                    kFThreads, st, false, mq, mk, mp, ma, prm, pk);
  return mask_bias ? launch_short(attn_qk_bsb_short_kernel<true, false>, tiles, kFSmem, kFThreads,
                                  st, false, mq, mk, mp, ma, prm, pk)
                   : launch_short(attn_qk_bsb_short_kernel<false, false>, tiles, kFSmem,
                                  kFThreads, st, false, mq, mk, mp, ma, prm, pk);
}

cudaError_t launch_attn_da_bsbb_short(int B, int H, int J, int P, float scale, const void* dC,
                                      int64_t lddc, const void* V, int64_t ldv, const void* Pin,
                                      const PhiloxKey& pk, int64_t batch_offset,
                                      const uint32_t* keep_bits, void* dS, cudaStream_t st,
                                      bool high_prio) {
  if (!attn_short_supported(J, P)) return cudaErrorInvalidValue;
  CUtensorMap mc, mv, mp, ms;
  bool ok = map_pop(&mc, dC, B, H, J, P, lddc, kS) && map_pop(&mv, V, B, H, J, P, ldv, kS) &&
            map_bhrc_s(&mp, Pin, B, H, J, J, 64, 32, CU_TENSOR_MAP_SWIZZLE_128B) &&
            map_bhrc_s(&ms, dS, B, H, J, J, 64, 32, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!ok) return cudaErrorInvalidValue;
  const int tiles = B * H;
  ShortParams prm{H,       tiles, scale, batch_offset * (int64_t)H * J * (J / 8),
                  nullptr, const_cast<uint32_t*>(keep_bits), 0, 0, 0};
  return launch_short(attn_da_bsbb_short_kernel, tiles, kBSmem, kBThreads, st, high_prio, mc, mv, mp, ms,
                      prm, pk);
}

}  // namespace enc

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
// Tile = one (b, h) pair x 128 query rows x all K = 512 keys: the fp32 score / gradient tile
// fills the 512 TMEM columns, so every row's softmax statistics are complete inside the
// CTA.  Persistent CTAs of 32 warps (one CTA per SM).  Every warp is an epilogue warp: warp
// w owns TMEM lane quarter q = w % 4 (rows 32q..32q+31) and the 64-column slice w / 4; the
// 8 slices of a row exchange row statistics through shared memory behind one named barrier
// per quarter.  Warp 0 lane 0 is also the TMA producer and tcgen05.mma issuer: between its
// epilogue tiles it issues the next tile's MMA (once all 32 warps released TMEM) and then
// the operand loads of the tile after.  32 warps per SM (8 per scheduler) hide the TMEM,
// MUFU and Philox latencies of the element-wise epilogue.
// Forward epilogue: pass 1 row max, pass 2 e = 2^(y - max) written back to TMEM + row sum
// (one MUFU.EX2 per element), pass 3 P = e / sum and A = dropout(P), staged per warp in a
// 64-B-swizzled [32 x 32] tile pair and written by TMA stores.
// Backward epilogue: each warp TMA-loads its own [32 x 64] P sub-tile (one tile ahead, its
// own mbarrier), pass 1 sum_k dropout(dA)*P with the keep bits kept in registers, pass 2
// dS written in place of the P sub-tile and stored by TMA.  With the forward's attention
// output C given (kDC, R26), the row term sum_k dP*P is the identity
// sum_p dC*C (C = A V, A = dropout(P)), formed from dC and C (fp32 as two bf16 words,
// C_hi by TMA with the operands) while the MMA runs: pass 1, its wait for P and its
// cross-warp barrier disappear and the epilogue is one pass over TMEM (measured at config L:
// 53 -> 45 us alone, 48 -> 39 us in the layer's graph).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include <type_traits>

#include "kernels.h"
#include "tc_gemm.cuh"

namespace enc {
namespace {

constexpr int kK = 512;             // keys per row (= J); the whole row lives in TMEM
constexpr int kRows = 128;          // query rows per tile (MMA M)
constexpr int kWarps = 32;
constexpr int kThreads = kWarps * 32;
constexpr int kSlices = kWarps / 4; // column slices per row
constexpr int kW = kK / kSlices;    // 64 columns per warp
constexpr float kL2e = 1.4426950408889634f;

struct FusedParams {
  int H, J;
  int tiles;        // (J / 128) * B * H
  float c;          // scale * log2(e)   (fwd)  |  scale  (bwd)
  int64_t g0;       // Philox chunk index of element (b=0,h=0,j=0,k=0) of this call
  const float* mask_bias;  // [B, K] or null (fwd)
  uint32_t* keep_bits;     // [B, H, J, K/32] keep-flag words (fwd: written if non-null;
                           // bwd: read instead of recomputing Philox when kBits)
  int write_a;             // fwd: A = dropout(P) stored (0: only P and the keep words)
  int keep_pre;            // fwd: keep_bits already hold this call's keep words (read them)
  // bwd kDC: dC and the forward's attention output C = C_hi + C_lo ([B,J,H,P] rows)
  const __nv_bfloat16* dc;
  const __nv_bfloat16* chi;
  const __nv_bfloat16* clo;
  int64_t ld_dc, ld_c;
};

__device__ __forceinline__ uint4 ld_nc4(const __nv_bfloat16* p) {
  uint4 v;
  asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void qbar(int q) {   // the 8 warps of TMEM lane quarter q
  asm volatile("bar.sync %0, %1;" ::"r"(1 + q), "r"(kSlices * 32) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ uint4 pack8(const float* v) {
  uint4 u;
  u.x = Chunk<__nv_bfloat16>::pack2(v[0], v[1]);
  u.y = Chunk<__nv_bfloat16>::pack2(v[2], v[3]);
  u.z = Chunk<__nv_bfloat16>::pack2(v[4], v[5]);
  u.w = Chunk<__nv_bfloat16>::pack2(v[6], v[7]);
  return u;
}

// mask-bias load kept in program order (volatile): hoisting all 64 loads above the MMA
// wait would spill
__device__ __forceinline__ float4 ld_mask4(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

// 16-B chunk c (0..3) of row r in a 64-B-row tile with the 64-byte TMA swizzle
__device__ __forceinline__ uint32_t sw64(int r, int c) {
  return (uint32_t)(r * 64 + ((c ^ ((r >> 1) & 3)) << 4));
}

// bit of element u (0..7) of chunk j (0..3) in a 32-element flag word
__device__ __forceinline__ constexpr int flag_bit(int j, int u) {
  return ((u & 1) ? 31 : 15) - (u >> 1) - 4 * j;
}

#ifdef ENC_FUSED_TRACE
// Debug-only phase timestamps (tools/trace_fused.py builds a separate library with this on).
__device__ unsigned long long g_fused_trace[148 * 2 * 8 * 8];
__device__ __forceinline__ void trace_ev(int warp, int lane, int it, int e) {
  if (lane == 0 && (warp == 0 || warp == 31) && it < 8 && blockIdx.x < 148) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_fused_trace[((blockIdx.x * 2 + (warp == 31)) * 8 + it) * 8 + e] = t;
  }
}
#define TRACE(e) trace_ev(warp, lane, it, (e))
#else
#define TRACE(e) ((void)0)
#endif

// shared-memory layout (bytes from a 1024-aligned base)
//   [0, 16K)     Q / dC tile [128 x 64] bf16 K-major SW128
//   [16K, 80K)   K / V  tile [512 x 64] bf16 K-major SW128 (two 256-row boxes)
//   [80K, 208K)  per-warp 4 KB regions: fwd staging ([32 x 32] P tile + A tile, SW64);
//                bwd the warp's [32 x 64] P sub-tile (SW128), overwritten in place by dS
//   then row statistics [2 parities][8 slices][128 rows] float2, barriers, tmem slot
constexpr uint32_t kOpA = 0, kOpB = 16384, kOpX = 81920;
constexpr uint32_t kStats = kOpX + kWarps * 4096;
constexpr uint32_t kBars = kStats + 2 * kSlices * kRows * 8;
constexpr uint32_t kLoX = kBars + 512;                     // bwd kDC: [2][4][32] float
constexpr size_t kSmem = 1024 + kLoX + 2 * 4 * 32 * 4;
static_assert(kSmem <= 227 * 1024, "smem");
static_assert(kW == 64, "two keep-flag words per thread");

template <bool kBwd, bool kMask, bool kBits, bool kCausal = false, bool kDC = false>
__device__ __forceinline__ void fused_body(const CUtensorMap& mapA, const CUtensorMap& mapB,
                                           const CUtensorMap& mapP, const CUtensorMap& mapO1,
                                           const CUtensorMap& mapO2, const FusedParams& prm,
                                           const PhiloxKey& pk, unsigned char* base,
                                           const CUtensorMap* mapC = nullptr) {
  static_assert(!kDC || kBwd, "kDC is a backward variant");
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int q = warp & 3;             // TMEM lane quarter
  const int slice = warp >> 2;        // 0..7
  const int r = q * 32 + lane;        // row within the tile
  const int cb = slice * kW;          // first column of this warp
  const int mtiles = prm.J / kRows;
  const bool leader = (warp == 0 && lane == 0);
  const bool hiT = pk.T >= 0x8000u;
  const uint32_t C2 = (hiT ? 0x10000u - pk.T : 0x8000u - pk.T) * 0x10001u;
  const uint32_t X = hiT ? 0u : 0xFFFFFFFFu;

  float2* stats = reinterpret_cast<float2*>(base + kStats);   // [2][8][128]
  uint64_t* op_full = reinterpret_cast<uint64_t*>(base + kBars);
  uint64_t* op_empty = op_full + 1;
  uint64_t* tm_full = op_full + 2;
  uint64_t* tm_empty = op_full + 3;
  uint64_t* p_full = op_full + 4;                              // [32] (bwd, per warp)
  uint64_t* dbar = op_full + 4 + kWarps;                       // (kDC) [4 quarters][2]
  uint64_t* d_done = op_full + 12 + kWarps;                    // (kDC) dC / C_hi tiles read
  float* lo_x = reinterpret_cast<float*>(base + kLoX);         // (kDC) [2][4][32]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(op_full + 13 + kWarps);
  unsigned char* own = base + kOpX + warp * 4096;              // this warp's 4 KB region

  auto tile_coords = [&](int t, int& b, int& h, int& m0, int& bh) {
    bh = t / mtiles;
    m0 = (t - bh * mtiles) * kRows;
    b = bh / prm.H;
    h = bh - b * prm.H;
  };
  auto load_operands = [&](int t) {
    int b, h, m0, bh;
    tile_coords(t, b, h, m0, bh);
    mbar_arrive_expect_tx(op_full, (uint32_t)(kRows + kK + (kDC ? kRows : 0)) * 128);
    if (kDC) tc::tma_load_4d(base + kStats, mapC, op_full, 0, h, m0, b);   // C_hi rows m0..
    // P-wide operand maps (map_pop): coordinates (p, h, row, b)
    tc::tma_load_4d(base + kOpA, &mapA, op_full, 0, h, m0, b);          // Q / dC rows m0..
    tc::tma_load_4d(base + kOpB, &mapB, op_full, 0, h, 0, b);           // K or V rows 0..255
    tc::tma_load_4d(base + kOpB + 256 * 128, &mapB, op_full, 0, h, 256, b);
  };
  auto load_psub = [&](int t) {      // bwd: this warp's [32 x 64] P sub-tile of tile t
    int b, h, m0, bh;
    tile_coords(t, b, h, m0, bh);
    mbar_arrive_expect_tx(&p_full[warp], 4096);
    tc::tma_load_4d(own, &mapP, &p_full[warp], cb, m0 + q * 32, h, b);
  };

  if (leader) {
    tc::prefetch_tmap(&mapA);
    tc::prefetch_tmap(&mapB);
    tc::prefetch_tmap(&mapO1);
    if (kBwd) tc::prefetch_tmap(&mapP);
    if (!kBwd) tc::prefetch_tmap(&mapO2);
    if (kDC) tc::prefetch_tmap(mapC);
    mbar_init(op_full, 1);
    mbar_init(op_empty, 1);
    mbar_init(tm_full, 1);
    mbar_init(tm_empty, kWarps);
    if (kDC) {
      for (int i = 0; i < 8; ++i) mbar_init(&dbar[i], kSlices * 32);
      mbar_init(d_done, kWarps);
    }
    fence_mbar_init();
  }
  if (kBwd && lane == 0) {
    mbar_init(&p_full[warp], 1);
    fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, kK);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16) + cb;
  pdl_wait();   // operands are the stream predecessor's outputs

  if (leader && blockIdx.x < prm.tiles) load_operands(blockIdx.x);
  if (kBwd && lane == 0 && blockIdx.x < prm.tiles) load_psub(blockIdx.x);
  int it = 0;
  for (int t = blockIdx.x; t < prm.tiles; t += gridDim.x, ++it) {
    int b, h, m0, bh;
    tile_coords(t, b, h, m0, bh);
    TRACE(0);
    if (leader) {
      // MMA of this tile once every warp released TMEM and the operands landed
      mbar_wait(tm_empty, (it & 1) ^ 1);
      mbar_wait(op_full, it & 1);
      tc::fence_after_sync();
      constexpr uint32_t idesc = tc::instr_desc_bf16_f32(kRows, 256, false, false);
      const uint64_t ad = tc::smem_desc(smem_u32(base + kOpA), 16, 1024);
      const uint64_t bd = tc::smem_desc(smem_u32(base + kOpB), 16, 1024);
#pragma unroll
      for (int nh = 0; nh < 2; ++nh)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc::mma_bf16(tmem + nh * 256, tc::desc_adv(ad, k * 32),
                       tc::desc_adv(bd, nh * 256 * 128 + k * 32), idesc, k != 0);
      tc::mma_commit(tm_full);
      tc::mma_commit(op_empty);
    }
    __syncwarp();
    // keep flags of this thread's 64 elements while the MMA runs (data independent):
    // recomputed from Philox, or (bwd) read back from the forward's keep-bit words
    const int64_t rowi = (int64_t)bh * prm.J + m0 + r;
    uint32_t kf[kW / 32];
    uint32_t* kbw = prm.keep_bits + rowi * (kK / 32) + cb / 32;
    if (kBits && (kBwd || prm.keep_pre)) {
      const uint2 w2 = __ldcs(reinterpret_cast<const uint2*>(kbw));
      kf[0] = w2.x;
      kf[1] = w2.y;
    } else if (pk.T == 0 || (!kBwd && !kBits && !prm.write_a)) {
      // p = 0: everything kept, no Philox stream.  Forward with neither A nor keep words
      // stored (the layer's path: A.V generates the mask on load, R28): the flags are unused
      kf[0] = kf[1] = 0xFFFFFFFFu;
      if (!kBwd && kBits) __stcs(reinterpret_cast<uint2*>(kbw), make_uint2(kf[0], kf[1]));
    } else {
      const int64_t grow = prm.g0 + rowi * (kK / 8) + cb / 8;
#pragma unroll
      for (int c = 0; c < kW / 32; ++c) {
        uint32_t f = 0;
#pragma unroll 2   // two Philox calls in flight: more would spill at 64 registers
        for (int j = 0; j < 4; ++j)
          f |= keep_flags((uint64_t)(grow + 4 * c + j), pk, C2, X, 4 * j);
        kf[c] = f;
      }
      if (!kBwd && kBits) __stcs(reinterpret_cast<uint2*>(kbw), make_uint2(kf[0], kf[1]));
    }
    TRACE(1);
    float Dc = 0.f;
    if constexpr (kDC) {
      // D_r = sum_p dC[r,p] (C_hi[r,p] + C_lo[r,p]).  C_hi part: per thread over its whole row
      // from the dC and C_hi tiles in shared memory.  C_lo part (a 2^-9 correction): warp
      // (q, s) forms it for rows 32q + 4s .. +3 from ONE coalesced 16-B load per lane (lane l:
      // row 4s + l/8, p-chunk l%8; issued before the C_hi part, which covers its latency), a
      // 3-step shuffle reduction over the row's 8 lanes, and hands the 4 sums to the quarter
      // through lo_x behind the quarter's per-parity mbarrier (read before pass 2)
      const int lrow = m0 + q * 32 + 4 * slice + (lane >> 3);
      const uint4 ul = ld_nc4(prm.clo + ((int64_t)b * prm.J + lrow) * prm.ld_c + h * 64 +
                              (lane & 7) * 8);
      mbar_wait(op_full, it & 1);
      float dacc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        float x[8], y[8];
        Chunk<__nv_bfloat16>::unpack(
            *reinterpret_cast<const uint4*>(base + kOpA + tc::sw128(r, c)), x);
        Chunk<__nv_bfloat16>::unpack(
            *reinterpret_cast<const uint4*>(base + kStats + tc::sw128(r, c)), y);
#pragma unroll
        for (int u = 0; u < 8; ++u) dacc[u & 3] = fmaf(x[u], y[u], dacc[u & 3]);
      }
      Dc = (dacc[0] + dacc[1]) + (dacc[2] + dacc[3]);
      {
        float xd[8], xl[8];
        Chunk<__nv_bfloat16>::unpack(*reinterpret_cast<const uint4*>(
                                         base + kOpA + tc::sw128(lrow - m0, lane & 7)), xd);
        Chunk<__nv_bfloat16>::unpack(ul, xl);
        float part = 0.f;
#pragma unroll
        for (int u = 0; u < 8; ++u) part = fmaf(xd[u], xl[u], part);
        part += __shfl_xor_sync(0xFFFFFFFFu, part, 1);
        part += __shfl_xor_sync(0xFFFFFFFFu, part, 2);
        part += __shfl_xor_sync(0xFFFFFFFFu, part, 4);
        if ((lane & 7) == 0) lo_x[((it & 1) * 4 + q) * 32 + 4 * slice + (lane >> 3)] = part;
        mbar_arrive(&dbar[q * 2 + (it & 1)]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(d_done);
    }
    mbar_wait_sleep(tm_full, it & 1);
    tc::fence_after_sync();
    TRACE(2);
    if (leader && t + (int)gridDim.x < prm.tiles) {   // operands free: prefetch the next tile
      mbar_wait(op_empty, it & 1);
      if (kDC) mbar_wait(d_done, it & 1);   // every warp has read dC and C_hi
      load_operands(t + gridDim.x);
    }
    float v[32];
    if (!kBwd) {
      // pass 1: per sub-chunk of kSub columns, y = scale*log2e*S (+ mask), sub-chunk max
      // m_c, e = 2^(y - m_c) back into TMEM, sub-chunk sum l_c.  The masked variant works
      // on 16 columns at a time (the mask values would otherwise spill at 64 registers).
      constexpr int kSub = kMask ? 16 : 32;
      constexpr int kNs = kW / kSub;
      const float c = prm.c;
      float mc[kNs], lc[kNs];
#pragma unroll
      for (int ch = 0; ch < kNs; ++ch) {
        float m;
        if (kMask) {
          tc::tmem_ld16(trow + ch * kSub, v);
          const float4* mb4 =
              reinterpret_cast<const float4*>(prm.mask_bias + (int64_t)b * kK + cb + ch * kSub);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float4 mm = ld_mask4(mb4 + i);
            v[4 * i + 0] = fmaf(v[4 * i + 0], c, mm.x * kL2e);
            v[4 * i + 1] = fmaf(v[4 * i + 1], c, mm.y * kL2e);
            v[4 * i + 2] = fmaf(v[4 * i + 2], c, mm.z * kL2e);
            v[4 * i + 3] = fmaf(v[4 * i + 3], c, mm.w * kL2e);
          }
          if (kCausal) {   // keys after the query row are masked out
#pragma unroll
            for (int i = 0; i < kSub; ++i)
              if (cb + ch * kSub + i > m0 + r) v[i] = -INFINITY;
          }
          m = tree_max<kSub>(v);
          const float mr = m == -INFINITY ? 0.f : m;
#pragma unroll
          for (int i = 0; i < kSub; ++i) v[i] = tc::ex2(v[i] - mr);
          lc[ch] = tree_sum<kSub>(v);
          tc::tmem_st16(trow + ch * kSub, v);
        } else {
          tc::tmem_ld32(trow + ch * kSub, v);
          if (kCausal) {   // keys after the query row are masked out
#pragma unroll
            for (int i = 0; i < kSub; ++i)
              if (cb + ch * kSub + i > m0 + r) v[i] = -INFINITY;
          }
          m = tree_max<kSub>(v) * c;   // c > 0
          // a fully masked chunk (causal) has m = -inf: exponentiate against 0 instead
          const float mz = (kCausal && m == -INFINITY) ? 0.f : m;
#pragma unroll
          for (int i = 0; i < kSub; ++i) v[i] = tc::ex2(fmaf(v[i], c, -mz));
          lc[ch] = tree_sum<kSub>(v);
          tc::tmem_st32(trow + ch * kSub, v);
        }
        mc[ch] = m;
      }
      float mt = mc[0];
#pragma unroll
      for (int ch = 1; ch < kNs; ++ch) mt = fmaxf(mt, mc[ch]);
      const float mtr = mt == -INFINITY ? 0.f : mt;
      float lt = 0.f;
#pragma unroll
      for (int ch = 0; ch < kNs; ++ch) lt += lc[ch] * tc::ex2(mc[ch] - mtr);
      float2* st = stats + (it & 1) * (kSlices * kRows);
      st[slice * kRows + r] = make_float2(mt, lt);
      tc::tmem_wait_st();
      TRACE(3);
      qbar(q);
      TRACE(4);
      // row max M and sum L over the 8 slices
      float M = st[r].x;
#pragma unroll
      for (int s2 = 1; s2 < kSlices; ++s2) M = fmaxf(M, st[s2 * kRows + r].x);
      const float Mr = M == -INFINITY ? 0.f : M;
      float L = 0.f;
#pragma unroll
      for (int s2 = 0; s2 < kSlices; ++s2) {
        const float2 x = st[s2 * kRows + r];
        L += x.y * tc::ex2(x.x - Mr);
      }
      const float invL = __fdividef(1.f, L);
      const float ds = pk.scale;
      // pass 2: P = e * 2^(m_c - M) / L and A = keep ? P * scale : 0, through the staging
      // pair, 32 columns per round
      float fP[kNs];
#pragma unroll
      for (int ch = 0; ch < kNs; ++ch) fP[ch] = tc::ex2(mc[ch] - Mr) * invL;
      // A not stored (the layer's path): the warp's whole [32 x 64] P sub-tile is staged in
      // its 4 KB region (128-B rows, SWIZZLE_128B) and leaves in ONE TMA store of full lines
      const bool p_only = !prm.write_a;
      if (p_only) {
        if (lane == 0) tc::bulk_wait_read<0>();   // the previous tile's store has read it
        __syncwarp();
      }
#pragma unroll
      for (int ch = 0; ch < kW / 32; ++ch) {
        if (!p_only) {
          if (lane == 0) tc::bulk_wait_read<0>();   // staging free again
          __syncwarp();
        }
        tc::tmem_ld32(trow + ch * 32, v);
        if (ch + 1 == kW / 32) {   // last TMEM read of this tile by this warp
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) mbar_arrive(tm_empty);
        }
        const uint32_t f = kf[ch];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float x[8], a[8];
          const float fp = fP[(ch * 32 + 8 * j) / kSub], fa = fp * ds;
#pragma unroll
          for (int u = 0; u < 8; ++u) x[u] = v[8 * j + u] * fp;
          if (p_only) {
            *reinterpret_cast<uint4*>(own + tc::sw128(lane, ch * 4 + j)) = pack8(x);
            continue;
          }
          *reinterpret_cast<uint4*>(own + sw64(lane, j)) = pack8(x);
          if (prm.write_a) {
#pragma unroll
            for (int u = 0; u < 8; ++u)
              a[u] = ((f >> flag_bit(j, u)) & 1u) ? v[8 * j + u] * fa : 0.f;
            *reinterpret_cast<uint4*>(own + 2048 + sw64(lane, j)) = pack8(a);
          }
        }
        if (p_only) continue;
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tc::tma_store_4d(&mapO1, own, cb + ch * 32, m0 + q * 32, h, b);
          if (prm.write_a) tc::tma_store_4d(&mapO2, own + 2048, cb + ch * 32, m0 + q * 32, h, b);
          tc::bulk_commit();
        }
      }
      if (p_only) {
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tc::tma_store_4d(&mapO2, own, cb, m0 + q * 32, h, b);   // P with 64-column boxes
          tc::bulk_commit();
        }
      }
      TRACE(5);
    } else {
      mbar_wait_sleep(&p_full[warp], it & 1);
      TRACE(3);
      // dS = scale * P * (dP - D'),  dP = keep ? sc * dA : 0,  D' = sc * dot
      const float ss = prm.c * pk.scale;        // scale * dropout scale
      float nDs;                                // -scale * D'
      if constexpr (kDC) {
        mbar_wait(&dbar[q * 2 + (it & 1)], (it >> 1) & 1);
        nDs = -(Dc + lo_x[((it & 1) * 4 + q) * 32 + lane]) * prm.c;   // D' includes sc
      } else {
        // pass 1: dot = sum_k keep_k * dA_k * P_k over this slice (x dropout scale below)
        float dacc[4] = {0.f, 0.f, 0.f, 0.f};   // four partial sums
#pragma unroll
        for (int ch = 0; ch < kW / 32; ++ch) {
          tc::tmem_ld32(trow + ch * 32, v);
          const uint32_t f = kf[ch];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float p[8];
            Chunk<__nv_bfloat16>::unpack(
                *reinterpret_cast<const uint4*>(own + tc::sw128(lane, ch * 4 + j)), p);
#pragma unroll
            for (int u = 0; u < 8; ++u)
              dacc[u & 3] = fmaf(((f >> flag_bit(j, u)) & 1u) ? v[8 * j + u] : 0.f, p[u],
                                 dacc[u & 3]);
          }
        }
        const float dot = (dacc[0] + dacc[1]) + (dacc[2] + dacc[3]);
        // row statistics alternate between the .x / .y slots by tile parity: a slot is
        // rewritten two tiles later, after every warp of the quarter passed the next barrier
        float* st = reinterpret_cast<float*>(stats) + (it & 1);
        st[2 * (slice * kRows + r)] = dot;
        TRACE(4);
        qbar(q);
        TRACE(5);
        float D = 0.f;
#pragma unroll
        for (int s2 = 0; s2 < kSlices; ++s2) D += st[2 * (s2 * kRows + r)];
        nDs = -D * ss;
      }
      // pass 2: dS over the P sub-tile in place
#pragma unroll
      for (int ch = 0; ch < kW / 32; ++ch) {
        tc::tmem_ld32(trow + ch * 32, v);
        if (ch + 1 == kW / 32) {
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) mbar_arrive(tm_empty);
        }
        const uint32_t f = kf[ch];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float p[8];
          uint4* loc = reinterpret_cast<uint4*>(own + tc::sw128(lane, ch * 4 + j));
          Chunk<__nv_bfloat16>::unpack(*loc, p);
#pragma unroll
          for (int u = 0; u < 8; ++u)
            p[u] *= ((f >> flag_bit(j, u)) & 1u) ? fmaf(v[8 * j + u], ss, nDs) : nDs;
          *loc = pack8(p);
        }
      }
      TRACE(6);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tc::tma_store_4d(&mapO1, own, cb, m0 + q * 32, h, b);
        tc::bulk_commit();
        // the next tile's P sub-tile may land here once the store has read it
        if (t + (int)gridDim.x < prm.tiles) {
          tc::bulk_wait_read<0>();
          load_psub(t + gridDim.x);
        }
      }
      __syncwarp();
      TRACE(7);
    }
  }
  if (lane == 0) tc::bulk_wait<0>();
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, kK);
}

// ------------------------------------------------------------------ score kernel + A.V
// (R30) QK^T + BSB + A.V in one kernel: after the softmax the warp's P sub-tile is
// staged in shared memory (and stored, the backward needs P), dropout is applied to the staged
// values and the result A = keep * P (bf16) is written into TMEM over the consumed scores
// (columns [0, 256): 32 per slice, two keys per column) -- the A operand of
// C = A V (tcgen05.mma with A in TMEM), accumulated into columns [256, 320).  Warps 24-31
// read C out (x dropout scale) and store C and its low bf16 word (R26).  P is never re-read
// from HBM for the forward and the separate A.V launch disappears.
//   shared memory: Q [128 x 64] | K or V slot [512 x 64] | per-warp 4 KB staging | stats |
//   barriers.  The slot holds K from the previous tile's C = A V (c_full) to this tile's score
//   MMA (op_empty), then V: the next K never waits for this tile's P stores to drain.
__device__ __forceinline__ uint32_t half_mask2(uint32_t g) {   // bits 15 / 31 -> half masks
  uint32_t m;
  asm("prmt.b32 %0, %1, 0, 0xBB99;" : "=r"(m) : "r"(g));
  return m;
}

__device__ __forceinline__ void mma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

constexpr uint32_t kAvQ = 0, kAvV = 16384, kAvX = 81920;
constexpr uint32_t kAvStats = kAvX + kWarps * 4096;
constexpr uint32_t kAvBars = kAvStats + 2 * kSlices * kRows * 8;
constexpr size_t kAvSmem = 1024 + kAvBars + 16 * 8 + 16;
static_assert(kAvSmem <= 227 * 1024, "smem");

template <bool kMask, bool kCausal>
__global__ void __launch_bounds__(kThreads, 1) attn_qk_bsb_av_kernel(
    const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapK,
    const __grid_constant__ CUtensorMap mapV, const __grid_constant__ CUtensorMap mapP,
    const __grid_constant__ CUtensorMap mapC, const __grid_constant__ CUtensorMap mapClo,
    FusedParams prm, PhiloxKey pk) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = tc::align1024(smem_raw);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int q = warp & 3;
  const int slice = warp >> 2;
  const int r = q * 32 + lane;
  const int cb = slice * kW;
  const int mtiles = prm.J / kRows;
  const bool leader = (warp == 0 && lane == 0);
  const bool hiT = pk.T >= 0x8000u;
  const uint32_t C2 = (hiT ? 0x10000u - pk.T : 0x8000u - pk.T) * 0x10001u;
  const uint32_t X = hiT ? 0u : 0xFFFFFFFFu;

  float2* stats = reinterpret_cast<float2*>(base + kAvStats);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + kAvBars);
  uint64_t* op_full = bars + 0;    // Q + K landed (count 2: Q and K are issued separately)
  uint64_t* op_empty = bars + 1;   // score MMA done (Q slot free, the K in the V slot read)
  uint64_t* tm_full = bars + 2;    // S in TMEM
  uint64_t* s_read = bars + 3;     // every warp read its S columns (count 32)
  uint64_t* a_ready = bars + 4;    // every warp wrote its A columns (count 32)
  uint64_t* v_full = bars + 5;     // V landed
  uint64_t* c_full = bars + 6;     // C = A V in TMEM (also: V slot and A columns free)
  uint64_t* c_done = bars + 7;     // C read out of TMEM (count 8)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 9);
  unsigned char* own = base + kAvX + warp * 4096;

  auto tile_coords = [&](int t, int& b, int& h, int& m0, int& bh) {
    bh = t / mtiles;
    m0 = (t - bh * mtiles) * kRows;
    b = bh / prm.H;
    h = bh - b * prm.H;
  };
  // the V slot holds K from the previous tile's C = A V until this tile's score MMA, then V:
  // K never waits for the P stores to drain out of the staging
  auto load_q = [&](int t) {
    int b, h, m0, bh;
    tile_coords(t, b, h, m0, bh);
    mbar_arrive_expect_tx(op_full, (uint32_t)kRows * 128);
    tc::tma_load_4d(base + kAvQ, &mapQ, op_full, 0, h, m0, b);
  };
  auto load_k = [&](int t) {
    int b, h, m0, bh;
    tile_coords(t, b, h, m0, bh);
    mbar_arrive_expect_tx(op_full, (uint32_t)kK * 128);
    tc::tma_load_4d(base + kAvV, &mapK, op_full, 0, h, 0, b);
    tc::tma_load_4d(base + kAvV + 256 * 128, &mapK, op_full, 0, h, 256, b);
  };
  auto load_v = [&](int t) {
    int b, h, m0, bh;
    tile_coords(t, b, h, m0, bh);
    mbar_arrive_expect_tx(v_full, (uint32_t)kK * 128);
    tc::tma_load_4d(base + kAvV, &mapV, v_full, 0, h, 0, b);
    tc::tma_load_4d(base + kAvV + 256 * 128, &mapV, v_full, 0, h, 256, b);
  };

  if (leader) {
    tc::prefetch_tmap(&mapQ);
    tc::prefetch_tmap(&mapK);
    tc::prefetch_tmap(&mapV);
    tc::prefetch_tmap(&mapP);
    tc::prefetch_tmap(&mapC);
    tc::prefetch_tmap(&mapClo);
    mbar_init(op_full, 2);
    mbar_init(op_empty, 1);
    mbar_init(tm_full, 1);
    mbar_init(s_read, kWarps);
    mbar_init(a_ready, kWarps);
    mbar_init(v_full, 1);
    mbar_init(c_full, 1);
    mbar_init(c_done, 8);
    fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, kK);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16) + cb;
  pdl_wait();   // operands are the stream predecessor's outputs

  if (leader && blockIdx.x < prm.tiles) {
    load_q(blockIdx.x);
    load_k(blockIdx.x);
  }

  // keep flags of this thread's 64 elements of tile tt (needed: A = keep * P) and the keep
  // words for the backward
  auto draw_flags = [&](int tt, uint32_t kf[2]) {
    int b2, h2, m2, bh2;
    tile_coords(tt, b2, h2, m2, bh2);
    const int64_t rowi = (int64_t)bh2 * prm.J + m2 + r;
    if (pk.T == 0) {
      kf[0] = kf[1] = 0xFFFFFFFFu;
    } else {
      const int64_t grow = prm.g0 + rowi * (kK / 8) + cb / 8;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t f = 0;
#pragma unroll 2
        for (int j = 0; j < 4; ++j)
          f |= keep_flags((uint64_t)(grow + 4 * c + j), pk, C2, X, 4 * j);
        kf[c] = f;
      }
    }
    __stcs(reinterpret_cast<uint2*>(prm.keep_bits + rowi * (kK / 32) + cb / 32),
           make_uint2(kf[0], kf[1]));
  };
  // C = A V is issued by a C read-out warp (idle until C is ready anyway): warp 0, which
  // issues the score MMAs, goes on to the next tile's flags as soon as its A is written
  const bool av_issuer = warp == 24 && lane == 0;

  int it = 0;
  uint32_t kf[2];
  for (int t = blockIdx.x; t < prm.tiles; t += gridDim.x, ++it) {
    int b, h, m0, bh;
    tile_coords(t, b, h, m0, bh);
    const uint32_t ph = it & 1;
    TRACE(0);
    draw_flags(t, kf);
    TRACE(1);
    // (the MMA-issuing thread draws its flags first: issued earlier, its warp would enter
    // pass 1 a flag phase late and hold back its quarter)
    if (leader) {
      // score MMA once the previous tile's C left TMEM and this tile's Q, K landed
      if (it > 0) mbar_wait(c_done, ph ^ 1);
      mbar_wait(op_full, ph);
      tc::fence_after_sync();
      constexpr uint32_t idesc = tc::instr_desc_bf16_f32(kRows, 256, false, false);
      const uint64_t ad = tc::smem_desc(smem_u32(base + kAvQ), 16, 1024);
      const uint64_t bd = tc::smem_desc(smem_u32(base + kAvV), 16, 1024);
#pragma unroll
      for (int nh = 0; nh < 2; ++nh)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc::mma_bf16(tmem + nh * 256, tc::desc_adv(ad, k * 32),
                       tc::desc_adv(bd, nh * 256 * 128 + k * 32), idesc, k != 0);
      tc::mma_commit(tm_full);
      tc::mma_commit(op_empty);
    }
    __syncwarp();
    mbar_wait_sleep(tm_full, ph);
    tc::fence_after_sync();
    if (warp == 24 && lane == 0) {
      // the score MMA has read Q and K: this tile's V into the V slot, the next tile's Q
      mbar_wait(op_empty, ph);
      load_v(t);
      if (t + (int)gridDim.x < prm.tiles) load_q(t + gridDim.x);
    }
    TRACE(2);
    float v[32];
    // pass 1 (as fused_body): sub-chunk max, e = 2^(y - m_c) back into TMEM, sub-chunk sum
    constexpr int kSub = kMask ? 16 : 32;
    constexpr int kNs = kW / kSub;
    const float c = prm.c;
    float mc[kNs], lc[kNs];
#pragma unroll
    for (int ch = 0; ch < kNs; ++ch) {
      float m;
      if (kMask) {
        tc::tmem_ld16(trow + ch * kSub, v);
        const float4* mb4 =
            reinterpret_cast<const float4*>(prm.mask_bias + (int64_t)b * kK + cb + ch * kSub);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float4 mm = ld_mask4(mb4 + i);
          v[4 * i + 0] = fmaf(v[4 * i + 0], c, mm.x * kL2e);
          v[4 * i + 1] = fmaf(v[4 * i + 1], c, mm.y * kL2e);
          v[4 * i + 2] = fmaf(v[4 * i + 2], c, mm.z * kL2e);
          v[4 * i + 3] = fmaf(v[4 * i + 3], c, mm.w * kL2e);
        }
        if (kCausal) {
#pragma unroll
          for (int i = 0; i < kSub; ++i)
            if (cb + ch * kSub + i > m0 + r) v[i] = -INFINITY;
        }
        m = tree_max<kSub>(v);
        const float mr = m == -INFINITY ? 0.f : m;
#pragma unroll
        for (int i = 0; i < kSub; ++i) v[i] = tc::ex2(v[i] - mr);
        lc[ch] = tree_sum<kSub>(v);
        tc::tmem_st16(trow + ch * kSub, v);
      } else {
        tc::tmem_ld32(trow + ch * kSub, v);
        if (kCausal) {
#pragma unroll
          for (int i = 0; i < kSub; ++i)
            if (cb + ch * kSub + i > m0 + r) v[i] = -INFINITY;
        }
        m = tree_max<kSub>(v) * c;
        const float mz = (kCausal && m == -INFINITY) ? 0.f : m;
#pragma unroll
        for (int i = 0; i < kSub; ++i) v[i] = tc::ex2(fmaf(v[i], c, -mz));
        lc[ch] = tree_sum<kSub>(v);
        tc::tmem_st32(trow + ch * kSub, v);
      }
      mc[ch] = m;
    }
    float mt = mc[0];
#pragma unroll
    for (int ch = 1; ch < kNs; ++ch) mt = fmaxf(mt, mc[ch]);
    const float mtr = mt == -INFINITY ? 0.f : mt;
    float lt = 0.f;
#pragma unroll
    for (int ch = 0; ch < kNs; ++ch) lt += lc[ch] * tc::ex2(mc[ch] - mtr);
    float2* st = stats + (it & 1) * (kSlices * kRows);
    st[slice * kRows + r] = make_float2(mt, lt);
    tc::tmem_wait_st();
    qbar(q);
    TRACE(3);
    float M = st[r].x;
#pragma unroll
    for (int s2 = 1; s2 < kSlices; ++s2) M = fmaxf(M, st[s2 * kRows + r].x);
    const float Mr = M == -INFINITY ? 0.f : M;
    float L = 0.f;
#pragma unroll
    for (int s2 = 0; s2 < kSlices; ++s2) {
      const float2 x2 = st[s2 * kRows + r];
      L += x2.y * tc::ex2(x2.x - Mr);
    }
    const float invL = __fdividef(1.f, L);
    float fP[kNs];
#pragma unroll
    for (int ch = 0; ch < kNs; ++ch) fP[ch] = tc::ex2(mc[ch] - Mr) * invL;
    // pass 2: P staged as the warp's [32 x 64] SWIZZLE_128B tile (its previous contents --
    // P / C of the last tile -- have been read: see the bulk waits)
    if (lane == 0) tc::bulk_wait_read<0>();
    __syncwarp();
#pragma unroll
    for (int ch = 0; ch < kW / 32; ++ch) {
      tc::tmem_ld32(trow + ch * 32, v);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float x[8];
        const float fp = fP[(ch * 32 + 8 * j) / kSub];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = v[8 * j + u] * fp;
        *reinterpret_cast<uint4*>(own + tc::sw128(lane, ch * 4 + j)) = pack8(x);
      }
    }
    tc::fence_before_sync();
    __syncwarp();
    TRACE(4);
    if (lane == 0) mbar_arrive(s_read);   // this warp's S columns are consumed
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      tc::tma_store_4d(&mapP, own, cb, m0 + q * 32, h, b);
      tc::bulk_commit();
    }
    // A = keep * P into TMEM columns [32 * slice, +32) of this warp's lanes, once every warp
    // has read its scores (the columns overlap other slices' S); 16 columns at a time
    mbar_wait(s_read, ph);
    tc::fence_after_sync();
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      float af[16];
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) {
        const int cc = half * 4 + c4;
        uint4 x = *reinterpret_cast<const uint4*>(own + tc::sw128(lane, cc));
        const uint32_t f = kf[half];
        const int j = c4;
        af[4 * c4 + 0] = __uint_as_float(x.x & half_mask2(f << (4 * j + 0)));
        af[4 * c4 + 1] = __uint_as_float(x.y & half_mask2(f << (4 * j + 1)));
        af[4 * c4 + 2] = __uint_as_float(x.z & half_mask2(f << (4 * j + 2)));
        af[4 * c4 + 3] = __uint_as_float(x.w & half_mask2(f << (4 * j + 3)));
      }
      tc::tmem_st16(tmem + ((uint32_t)(q * 32) << 16) + 32 * slice + 16 * half, af);
    }
    tc::tmem_wait_st();
    tc::fence_before_sync();
    __syncwarp();
    if (lane == 0) mbar_arrive(a_ready);
    TRACE(5);
    if (av_issuer) {
      // C = A V: 32 k-steps of 16 keys, A from TMEM (8 columns each), V MN-major
      mbar_wait(a_ready, ph);
      mbar_wait(v_full, ph);
      tc::fence_after_sync();
      constexpr uint32_t idesc_av = tc::instr_desc_bf16_f32(kRows, 64, false, true);
      const uint64_t vd = tc::smem_desc(smem_u32(base + kAvV), 8192, 1024);
#pragma unroll
      for (int ks = 0; ks < kK / 16; ++ks)
        mma_bf16_ts(tmem + 256, tmem + 8 * ks, tc::desc_adv(vd, ks * 2048), idesc_av, ks != 0);
      tc::mma_commit(c_full);
    }
    __syncwarp();
    if (warp >= 24) {
      // C (x dropout scale) or its low bf16 word, [32 rows x 64] per warp
      mbar_wait_sleep(c_full, ph);
      tc::fence_after_sync();
      TRACE(7);
      // the V slot is free once the A.V MMA completed: the next tile's K
      if (warp == 24 && lane == 0 && t + (int)gridDim.x < prm.tiles) load_k(t + gridDim.x);
      if (lane == 0) tc::bulk_wait_read<0>();   // this warp's P store has read the staging
      __syncwarp();
      const bool lo = warp >= 28;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        float cv[32];
        tc::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + 256 + 32 * hh, cv);
        if (hh == 1) {
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) mbar_arrive(c_done);   // C read out of TMEM
        }
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
          float x[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float y = cv[8 * c4 + u] * pk.scale;
            x[u] = lo ? y - __bfloat162float(__float2bfloat16_rn(y)) : y;
          }
          *reinterpret_cast<uint4*>(own + tc::sw128(lane, hh * 4 + c4)) = pack8(x);
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tc::tma_store_4d(lo ? &mapClo : &mapC, own, 0, h, m0 + q * 32, b);
        tc::bulk_commit();
      }
    }
    TRACE(6);
  }
  if (lane == 0) tc::bulk_wait<0>();
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, kK);
}

template <bool kMask, bool kBits, bool kCausal = false>
__global__ void __launch_bounds__(kThreads, 1) attn_qk_bsb_kernel(
    const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapK,
    const __grid_constant__ CUtensorMap mapP, const __grid_constant__ CUtensorMap mapA,
    FusedParams prm, PhiloxKey pk) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  fused_body<false, kMask, kBits, kCausal>(mapQ, mapK, mapQ, mapP, mapA, prm, pk,
                                           tc::align1024(smem_raw));
}

template <bool kBits, bool kDC>
__global__ void __launch_bounds__(kThreads, 1) attn_da_bsbb_kernel(
    const __grid_constant__ CUtensorMap mapdC, const __grid_constant__ CUtensorMap mapV,
    const __grid_constant__ CUtensorMap mapP, const __grid_constant__ CUtensorMap mapdS,
    FusedParams prm, PhiloxKey pk, const __grid_constant__ CUtensorMap mapC) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  fused_body<true, false, kBits, false, kDC>(mapdC, mapV, mapP, mapdS, mapdS, prm, pk,
                                             tc::align1024(smem_raw), &mapC);
}

bool map4(CUtensorMap* m, const void* ptr, const uint64_t d[4], const uint64_t s[3],
          const uint32_t box[4], CUtensorMapSwizzle sw) {
  cuuint64_t gdim[4] = {d[0], d[1], d[2], d[3]};
  cuuint64_t gstr[3] = {s[0] * 2, s[1] * 2, s[2] * 2};
  cuuint32_t bdim[4] = {box[0], box[1], box[2], box[3]};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return tmap_encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), gdim,
                           gstr, bdim, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// [B][H][rows][cols] with box {box_cols, box_rows}
bool map_bhrc(CUtensorMap* m, const void* p, int B, int H, int rows, int cols, int box_cols,
              int box_rows, CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  const uint64_t d[4] = {(uint64_t)cols, (uint64_t)rows, (uint64_t)H, (uint64_t)B};
  const uint64_t s[3] = {(uint64_t)cols, (uint64_t)rows * cols, (uint64_t)H * rows * cols};
  const uint32_t box[4] = {(uint32_t)box_cols, (uint32_t)box_rows, 1, 1};
  return map4(m, p, d, s, box, sw);
}

int persistent_grid(int tiles) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms <= 0) sms = 148;
  return tiles < sms ? tiles : sms;
}
}  // namespace

// the fewest CTAs that still finish `tiles` in the same number of waves as one CTA per SM
// (512 tiles on 148 SMs: 128 CTAs x 4 tiles -- the 20 SMs left over take side work, R31)
int balanced_grid(int tiles) {
  const int sms = persistent_grid(1 << 30);
  if (tiles <= 0) return 1;
  const int waves = (tiles + sms - 1) / sms;
  return (tiles + waves - 1) / waves;
}

namespace {

template <typename Kern>
cudaError_t launch_persistent(Kern kern, int tiles, const CUtensorMap& a, const CUtensorMap& b,
                              const CUtensorMap& c, const CUtensorMap& d, const FusedParams& prm,
                              const PhiloxKey& pk, cudaStream_t st, bool high_prio = false,
                              const CUtensorMap* e = nullptr) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(persistent_grid(tiles));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (high_prio) {
    // the persistent kernel assumes all of its CTAs are resident at once: when a kernel on
    // another stream is ready at the same moment (the layer's dV beside the fused backward),
    // the block scheduler must place this one's CTAs first
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
  if constexpr (std::is_invocable_v<Kern, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap,
                                    FusedParams, PhiloxKey, CUtensorMap>)
    return cudaLaunchKernelEx(&cfg, kern, a, b, c, d, prm, pk, *e);
  else
    return cudaLaunchKernelEx(&cfg, kern, a, b, c, d, prm, pk);
}

// The attention keep words (ENC_KEEP_BITS layout) of a [B,H,J,K] call: one thread per 64
// columns (two words, eight Philox4x32-10 calls).  Launched ahead of the fused forward --
// in the layer on a side stream beside the QKV contraction, whose tensor-bound tiles leave
// the FMA pipe idle -- so the score kernel reads the words instead of running Philox
// between its MMA and its epilogue.
__global__ void __launch_bounds__(128) keep_bits_kernel(uint32_t* __restrict__ keep_bits,
                                                        int64_t n2, int K, int64_t g0,
                                                        PhiloxKey pk) {
  const bool hiT = pk.T >= 0x8000u;
  const uint32_t C2 = (hiT ? 0x10000u - pk.T : 0x8000u - pk.T) * 0x10001u;
  const uint32_t X = hiT ? 0u : 0xFFFFFFFFu;
  const int w2r = K / 64;   // word pairs per row
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rowi = i / w2r;
    const int cb = (int)(i - rowi * w2r) * 64;
    const int64_t grow = g0 + rowi * (K / 8) + cb / 8;
    uint32_t kf[2];
    if (pk.T == 0) {
      kf[0] = kf[1] = 0xFFFFFFFFu;
    } else {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t f = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) f |= keep_flags((uint64_t)(grow + 4 * c + j), pk, C2, X, 4 * j);
        kf[c] = f;
      }
    }
    __stcs(reinterpret_cast<uint2*>(keep_bits) + i, make_uint2(kf[0], kf[1]));
  }
}

}  // namespace

cudaError_t launch_attn_keep_bits(int B, int H, int J, int K, const PhiloxKey& pk,
                                  int64_t batch_offset, uint32_t* keep_bits, cudaStream_t st) {
  if (K % 64) return cudaErrorInvalidValue;
  const int64_t n2 = (int64_t)B * H * J * (K / 64);
  if (n2 == 0) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // one 128-thread block per SM: beside the persistent QKV contraction (1 CTA per SM, 96
  // registers x 576 threads) a block of 128 x 30 registers still fits, so the two overlap
  // whichever is placed first
  int64_t grid = (n2 + 127) / 128;
  if (grid > 2 * sms) grid = 2 * sms;
  keep_bits_kernel<<<(int)grid, 128, 0, st>>>(keep_bits, n2, K,
                                              batch_offset * (int64_t)H * J * (K / 8), pk);
  return cudaGetLastError();
}

// K = J = 512 (the whole score row in the 512 TMEM columns), or J = K = 128 (attn_short.cu),
// P = 64
bool attn_fused_supported(int J, int P) {
  return (P == 64 && J == kK) || attn_short_supported(J, P);
}

cudaError_t launch_attn_qk_bsb(int B, int H, int J, int P, float scale, const void* Q,
                               int64_t ldq, const void* Kt, int64_t ldk, const float* mask_bias,
                               const PhiloxKey& pk, int64_t batch_offset, void* Pout, void* Aout,
                               uint32_t* keep_bits, cudaStream_t st, int causal, int keep_pre,
                               bool high_prio) {
  if (attn_short_supported(J, P))
    return launch_attn_qk_bsb_short(B, H, J, P, scale, Q, ldq, Kt, ldk, mask_bias, pk,
                                    batch_offset, Pout, Aout, keep_bits, st, causal, keep_pre);
  const int K = J;
  CUtensorMap mq, mk, mp, ma;
  bool ok = map_pop(&mq, Q, B, H, J, P, ldq, kRows) && map_pop(&mk, Kt, B, H, K, P, ldk, 256) &&
            map_bhrc(&mp, Pout, B, H, J, K, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B) &&
            // A stored: A through 32-column boxes; else this map writes P in 64-column boxes
            (Aout ? map_bhrc(&ma, Aout, B, H, J, K, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B)
                  : map_bhrc(&ma, Pout, B, H, J, K, 64, 32));
  if (!ok) return cudaErrorInvalidValue;
  const int tiles = (J / kRows) * B * H;
  FusedParams prm{H,         J,         tiles, scale * kL2e, batch_offset * (int64_t)H * J * (K / 8),
                  mask_bias, keep_bits, Aout != nullptr, keep_pre && keep_bits ? 1 : 0};
  if (causal) {   // the masking step: keys k > j of each query row j removed
    if (mask_bias)
      return keep_bits ? launch_persistent(attn_qk_bsb_kernel<true, true, true>, tiles, mq, mk, mp,
                                           ma, prm, pk, st, high_prio)
                       : launch_persistent(attn_qk_bsb_kernel<true, false, true>, tiles, mq, mk,
                                           mp, ma, prm, pk, st, high_prio);
    return keep_bits ? launch_persistent(attn_qk_bsb_kernel<false, true, true>, tiles, mq, mk, mp,
                                         ma, prm, pk, st, high_prio)
                     : launch_persistent(attn_qk_bsb_kernel<false, false, true>, tiles, mq, mk,
                                         mp, ma, prm, pk, st, high_prio);
  }
  if (mask_bias)
    return keep_bits
               ? launch_persistent(attn_qk_bsb_kernel<true, true>, tiles, mq, mk, mp, ma, prm, pk, st, high_prio)
               : launch_persistent(attn_qk_bsb_kernel<true, false>, tiles, mq, mk, mp, ma, prm, pk, st, high_prio);
  return keep_bits
             ? launch_persistent(attn_qk_bsb_kernel<false, true>, tiles, mq, mk, mp, ma, prm, pk, st, high_prio)
             : launch_persistent(attn_qk_bsb_kernel<false, false>, tiles, mq, mk, mp, ma, prm, pk, st, high_prio);
}

// QK^T + BSB + A.V in one kernel (R30): J = K = 512, P = 64; writes P, the keep words, C
// ([B,J,H,P] rows, stride ldc) and C's low bf16 word (same layout)
bool attn_fused_av_supported(int J, int P) { return P == 64 && J == kK; }

cudaError_t launch_attn_qk_bsb_av(int B, int H, int J, int P, float scale, const void* Q,
                                  int64_t ldq, const void* Kt, int64_t ldk, const void* V,
                                  int64_t ldv, const float* mask_bias, const PhiloxKey& pk,
                                  int64_t batch_offset, void* Pout, uint32_t* keep_bits,
                                  void* C, void* C_lo, int64_t ldc, cudaStream_t st, int causal) {
  if (!attn_fused_av_supported(J, P) || !keep_bits || !C || !C_lo)
    return cudaErrorInvalidValue;
  const int K = J;
  CUtensorMap mq, mk, mv, mp, mc, ml;
  bool ok = map_pop(&mq, Q, B, H, J, P, ldq, kRows) && map_pop(&mk, Kt, B, H, K, P, ldk, 256) &&
            map_pop(&mv, V, B, H, K, P, ldv, 256) && map_bhrc(&mp, Pout, B, H, J, K, 64, 32) &&
            map_pop(&mc, C, B, H, J, P, ldc, 32) && map_pop(&ml, C_lo, B, H, J, P, ldc, 32);
  if (!ok) return cudaErrorInvalidValue;
  const int tiles = (J / kRows) * B * H;
  FusedParams prm{H,         J,         tiles, scale * kL2e, batch_offset * (int64_t)H * J * (K / 8),
                  mask_bias, keep_bits, 0, 0};
  auto go = [&](auto kern) -> cudaError_t {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kAvSmem);
    return launch_k(PDL_ATTN_FUSED, kern, balanced_grid(tiles), kThreads, kAvSmem, st, mq, mk,
                    mv, mp, mc, ml, prm, pk);
  };
  if (causal)
    return mask_bias ? go(attn_qk_bsb_av_kernel<true, true>) : go(attn_qk_bsb_av_kernel<false, true>);
  return mask_bias ? go(attn_qk_bsb_av_kernel<true, false>) : go(attn_qk_bsb_av_kernel<false, false>);
}

cudaError_t launch_attn_da_bsbb(int B, int H, int J, int P, float scale, const void* dC,
                                int64_t lddc, const void* V, int64_t ldv, const void* Pin,
                                const PhiloxKey& pk, int64_t batch_offset,
                                const uint32_t* keep_bits, void* dS, cudaStream_t st,
                                bool high_prio, const void* Chi, const void* Clo,
                                int64_t ldc) {
  if (attn_short_supported(J, P))
    return launch_attn_da_bsbb_short(B, H, J, P, scale, dC, lddc, V, ldv, Pin, pk, batch_offset,
                                     keep_bits, dS, st, high_prio);
  const int K = J;
  CUtensorMap mc, mv, mp, ms;
  bool ok = map_pop(&mc, dC, B, H, J, P, lddc, kRows) && map_pop(&mv, V, B, H, K, P, ldv, 256) &&
            map_bhrc(&mp, Pin, B, H, J, K, 64, 32) && map_bhrc(&ms, dS, B, H, J, K, 64, 32);
  if (!ok) return cudaErrorInvalidValue;
  const bool dc = Chi && Clo;
  if (dc && (((uintptr_t)dC | (uintptr_t)Chi | (uintptr_t)Clo) & 15u || lddc % 8 || ldc % 8))
    return cudaErrorInvalidValue;
  const int tiles = (J / kRows) * B * H;
  FusedParams prm{H,       J,       tiles, scale, batch_offset * (int64_t)H * J * (K / 8),
                  nullptr, const_cast<uint32_t*>(keep_bits), 0, 0,
                  (const __nv_bfloat16*)dC, (const __nv_bfloat16*)Chi,
                  (const __nv_bfloat16*)Clo, lddc, ldc};
  if (dc) {   // the C_hi tile arrives with the operands (C_lo is read by the warps)
    CUtensorMap mC;
    if (!map_pop(&mC, Chi, B, H, J, P, ldc, kRows)) return cudaErrorInvalidValue;
    return keep_bits ? launch_persistent(attn_da_bsbb_kernel<true, true>, tiles, mc, mv, mp, ms,
                                         prm, pk, st, high_prio, &mC)
                     : launch_persistent(attn_da_bsbb_kernel<false, true>, tiles, mc, mv, mp, ms,
                                         prm, pk, st, high_prio, &mC);
  }
  return keep_bits ? launch_persistent(attn_da_bsbb_kernel<true, false>, tiles, mc, mv, mp, ms,
                                       prm, pk, st, high_prio, &mc)
                   : launch_persistent(attn_da_bsbb_kernel<false, false>, tiles, mc, mv, mp, ms,
                                       prm, pk, st, high_prio, &mc);
}

#ifdef ENC_FUSED_TRACE
extern "C" int enc_debug_fused_trace(void* host, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(host, g_fused_trace, bytes);
}
extern "C" int enc_debug_fused_trace_clear() {
  static unsigned long long zero[148 * 2 * 8 * 8];
  return (int)cudaMemcpyToSymbol(g_fused_trace, zero, sizeof(zero));
}
#endif

}  // namespace enc

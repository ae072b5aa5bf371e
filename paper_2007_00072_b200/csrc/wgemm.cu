// Hand-written tcgen05 weight contractions of the encoder layer (Table A.1 contraction rows:
// Q,K,V PAPER.md:549, Out :554, Linear :559 / :563 forward; their dX / dW :573-574,
// :579-580, :586-587, :593-594), with the epilogue fusions the paper could not get from a
// library (it rejected CUTLASS epilogue fusion on V100):
//   EPI_STORE    C = A op B (+ fp32 bias over columns: AIB, :550) (+ C: the β = 1 residual of
//                `ebsb` :581 / `bei` :596), bf16 or fp32 output; split-K for fp32 outputs
//   EPI_BAD_FWD  Linear1 + BAD (`brd`): h = acc + b1 (stored, bf16),
//                A1 = dropout(act(h)) -- the Y1 round trip and the BAD launch disappear
//   EPI_BAD_BWD  Linear2-dX + BAD-bwd (`bdrb`): dh = dropout'(acc) ⊙
//                act'(h) with h read from the saved set, plus per-32-row column partials of
//                dh (db1) -- the dA1 round trip and the BAD-bwd launch disappear
//
// Row-major operands in nn.Linear convention: C[M,N] = A·B with
//   A K-major ([M][K], forward / dX) or MN-major ([K][M], dW = dYᵀ X),
//   B K-major ([N][K], forward: the weight) or MN-major ([K][N], dX: the weight; dW: X).
//
// Persistent, warp-specialised CTA (one per SM, 320 threads):
//   warp 0      TMA producer: 4-stage ring of 128x64 A and 256x64 B k-blocks (SWIZZLE_128B)
//   warp 1      TMEM allocator + MMA issuer: tcgen05.mma M=128 N=256 K=16, fp32 accumulator
//               double-buffered in TMEM (2 x 256 columns) so a tile's epilogue overlaps the
//               next tile's main loop
//   warps 2-9   epilogue: warp w reads TMEM lane quarter w % 4, column half (w-2)/4;
//               per 64-byte column chunk: tcgen05.ld -> fused math -> 64B-swizzled [32 x 64 B]
//               staging -> TMA store (double-buffered per warp); auxiliary inputs (h, the
//               residual) arrive by TMA into the same staging buffers one chunk ahead
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "act.cuh"
#include "kernels.h"
#include "tc_gemm.cuh"

namespace enc {
namespace wg {

#ifdef ENC_WGEMM_TRACE
// Debug-only timeline (tools/trace_wgemm.py builds a separate library with this on):
// per CTA and tile index (< 8): [0] MMA warp starts the tile (accumulator free),
// [1] its last MMA committed, [2] epilogue warp 2 has the accumulator, [3] it finished.
__device__ unsigned long long g_wg_trace[148 * 8 * 4];
__device__ __forceinline__ void wg_stamp(int it, int e) {
  if (it < 8 && blockIdx.x < 148) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_wg_trace[(blockIdx.x * 8 + it) * 4 + e] = t;
  }
}
#define WG_STAMP(it, e) wg_stamp((it), (e))
#else
#define WG_STAMP(it, e) ((void)0)
#endif


constexpr int kBM = 128, kBN = 256, kBK = 64;   // per-CTA accumulator tile 128 x 256
constexpr int kEpiWarps = 16;                   // 4 per TMEM lane quarter
constexpr int kSliceCols = kBN / (kEpiWarps / 4);  // accumulator columns per epilogue warp
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr uint32_t kABytes = kBM * kBK * 2;   // 16 KB per stage
constexpr uint32_t kStg = 32 * 64;            // one [32 rows x 64 B] staging buffer

// CG = 1: one CTA computes a 128 x 256 tile (tcgen05.mma.cta_group::1, M = 128, N = 256).
// CG = 2: a CTA pair (cluster of 2 on one TPC) computes a 256 x 256 tile with
// tcgen05.mma.cta_group::2 (M = 256, N = 256) issued by the even CTA: each CTA stages
// half of A (its 128 rows) and half of B (128 of the 256 columns) and holds its 128 rows x
// 256 columns of the accumulator, so per-SM shared-memory and L2 operand traffic per MMA
// drop by a third against CG = 1.
template <int CG, int EPI>
struct Cfg {
  static constexpr uint32_t kBBytes = (kBN / CG) * kBK * 2;
  static constexpr int kStages = CG == 2 ? 5 : 3;
  static constexpr int kNBuf = 2;   // staging buffers per epilogue warp
  static constexpr size_t kSmem = 1024 + (size_t)kStages * (kABytes + kBBytes) +
                                  (size_t)kEpiWarps * kNBuf * kStg + 256;
};

struct Params {
  int M, N, K;
  int tiles_m, tiles_n, splits, units;   // tiles of (128 CG) x 256; units = tiles x splits
  int kb_per_split, nk;
  int beta;               // EPI_STORE: out = acc (+ bias) + out (bf16 output)
  const float* bias;      // [N] fp32 or null (EPI_STORE, EPI_BAD_FWD: b1)
  PhiloxKey pk;           // BAD epilogues (site 2)
  int64_t g0;             // Philox chunk index of element (0, 0): batch_offset * J * N / 8
  float* partials;        // EPI_BAD_BWD: [ceil(M/128) * 4][N] column partial sums of dh
  uint8_t* kb_out;        // EPI_BAD_FWD: keep bytes [M][N/8] written (or null)
  const uint8_t* kb_in;   // EPI_BAD_BWD / EPI_BAD_FWD: keep bytes [M][N/8] read instead of
                          // Philox (or null)
};

// byte offset of 16-B chunk c (0..3) of row r in a [32 x 64 B] SWIZZLE_64B tile
__device__ __forceinline__ uint32_t sw64(int r, int c) {
  return (uint32_t)(r * 64 + ((c ^ ((r >> 1) & 3)) << 4));
}

__device__ __forceinline__ void unpack_bf16x8(uint4 u, float* v) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[2 * i] = __uint_as_float(w[i] << 16);
    v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}
__device__ __forceinline__ uint4 pack_bf16x8(const float* v) {
  uint4 u;
  u.x = Chunk<__nv_bfloat16>::pack2(v[0], v[1]);
  u.y = Chunk<__nv_bfloat16>::pack2(v[2], v[3]);
  u.z = Chunk<__nv_bfloat16>::pack2(v[4], v[5]);
  u.w = Chunk<__nv_bfloat16>::pack2(v[6], v[7]);
  return u;
}

// ---- cluster (CTA pair) helpers
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
// shared::cluster address of the same shared-memory offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t caddr) {
  // default (.release.cta) semantics: what must be ordered before the arrive is this warp's
  // tcgen05.ld of the accumulator, which tcgen05.fence::before_thread_sync covers
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(caddr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// TMA 2-D load into this CTA's shared memory completing on the pair leader's mbarrier
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map,
                                                 uint32_t bar_caddr, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(bar_caddr)
      : "memory");
}
__device__ __forceinline__ void mma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// arrive on the mbarrier at this offset in both CTAs of the pair when the pair's MMAs finish
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

// unit -> (m block, n block, split); m fastest so concurrent CTAs share B tiles in L2
__device__ __forceinline__ void decode(const Params& p, int u, int& mb, int& nb, int& sp) {
  const int t = u % (p.tiles_m * p.tiles_n);
  sp = u / (p.tiles_m * p.tiles_n);
  mb = t % p.tiles_m;
  nb = t / p.tiles_m;
}

template <int CG, int AMN, int BMN, int OUTF32, int EPI, int ACT>
__global__ void __launch_bounds__(kThreads, 1)
    wgemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                 const __grid_constant__ CUtensorMap mapC, const __grid_constant__ CUtensorMap mapC2,
                 const __grid_constant__ CUtensorMap mapX, const Params p) {
  using C = Cfg<CG, EPI>;
  constexpr int kStages = C::kStages;
  constexpr uint32_t kBBytes = C::kBBytes;
  constexpr int kNBuf = C::kNBuf;
  constexpr int kBNc = kBN / CG;                 // B columns staged by this CTA
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = tc::align1024(smem_raw);
  unsigned char* sA = base;
  unsigned char* sB = base + kStages * kABytes;
  unsigned char* sStg = sB + kStages * kBBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sStg + kEpiWarps * kNBuf * kStg);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* xbar = tempty + 2;                 // 2 per epilogue warp (auxiliary loads)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xbar + 2 * kEpiWarps);

  constexpr bool kAux = EPI == EPI_BAD_BWD;    // (+ p.beta at run time)
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_rank() : 0;   // 0 = the pair's MMA issuer
  const int cid = blockIdx.x / CG;             // persistent scheduler: one unit per pair
  const int ncl = gridDim.x / CG;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&mapA);
    tc::prefetch_tmap(&mapB);
    tc::prefetch_tmap(&mapC);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], kEpiWarps * CG);
    }
    for (int s = 0; s < 2 * kEpiWarps; ++s) mbar_init(&xbar[s], 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       smem_u32(tmem_slot))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      tc::tmem_alloc(tmem_slot, 512);
    }
  }
  tc::fence_before_sync();
  if (CG == 2)
    cluster_sync();
  else
    __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();   // the activations are the stream predecessor's outputs

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t pc = 0;
      for (int u = cid; u < p.units; u += ncl) {
        int mb, nb, sp;
        decode(p, u, mb, nb, sp);
        const int m0 = mb * kBM * CG + rank * kBM;       // this CTA's A rows
        const int n0 = nb * kBN + rank * kBNc;           // this CTA's B columns
        const int kb0 = sp * p.kb_per_split;
        const int kb1 = min(p.nk, kb0 + p.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb, ++pc) {
          const uint32_t s = pc % kStages;
          mbar_wait(&empty[s], ((pc / kStages) & 1) ^ 1);
          const int k0 = kb * kBK;
          if (CG == 1) {
            mbar_arrive_expect_tx(&full[s], kABytes + kBBytes);
            if (!AMN) {
              tc::tma_load_2d(sA + s * kABytes, &mapA, &full[s], k0, m0);
            } else {
#pragma unroll
              for (int j = 0; j < kBM / 64; ++j)
                tc::tma_load_2d(sA + s * kABytes + j * 8192, &mapA, &full[s], m0 + 64 * j, k0);
            }
            if (!BMN) {
              tc::tma_load_2d(sB + s * kBBytes, &mapB, &full[s], k0, n0);
            } else {
#pragma unroll
              for (int j = 0; j < kBNc / 64; ++j)
                tc::tma_load_2d(sB + s * kBBytes + j * 8192, &mapB, &full[s], n0 + 64 * j, k0);
            }
          } else {
            // both CTAs' loads complete on the leader's full barrier, which expects them all
            const uint32_t fb = mapa(&full[s], 0);
            if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * (kABytes + kBBytes));
            if (!AMN) {
              tma_load_2d_pair(sA + s * kABytes, &mapA, fb, k0, m0);
            } else {
#pragma unroll
              for (int j = 0; j < kBM / 64; ++j)
                tma_load_2d_pair(sA + s * kABytes + j * 8192, &mapA, fb, m0 + 64 * j, k0);
            }
            if (!BMN) {
              tma_load_2d_pair(sB + s * kBBytes, &mapB, fb, k0, n0);
            } else {
#pragma unroll
              for (int j = 0; j < kBNc / 64; ++j)
                tma_load_2d_pair(sB + s * kBBytes + j * 8192, &mapB, fb, n0 + 64 * j, k0);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (pair leader)
    if (rank == 0) {
      constexpr uint32_t idesc = tc::instr_desc_bf16_f32(kBM * CG, kBN, AMN, BMN);
      uint32_t pc = 0;
      int it = 0;
      for (int u = cid; u < p.units; u += ncl, ++it) {
        int mb, nb, sp;
        decode(p, u, mb, nb, sp);
        const int kb0 = sp * p.kb_per_split;
        const int kb1 = min(p.nk, kb0 + p.kb_per_split);
        const int as = it & 1;
        if (CG == 2)
          mbar_wait_cluster(&tempty[as], ((it >> 1) & 1) ^ 1);
        else
          mbar_wait(&tempty[as], ((it >> 1) & 1) ^ 1);
        tc::fence_after_sync();
        if (lane == 0) WG_STAMP(it, 0);
        const uint32_t dacc = tmem + as * kBN;
        for (int kb = kb0; kb < kb1; ++kb, ++pc) {
          const uint32_t s = pc % kStages;
          if (CG == 2)
            mbar_wait_cluster(&full[s], (pc / kStages) & 1);
          else
            mbar_wait(&full[s], (pc / kStages) & 1);
          tc::fence_after_sync();
          if (lane == 0) {
            const uint64_t ad0 = tc::smem_desc(smem_u32(sA + s * kABytes), AMN ? 8192 : 16, 1024);
            const uint64_t bd0 = tc::smem_desc(smem_u32(sB + s * kBBytes), BMN ? 8192 : 16, 1024);
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              const uint64_t ad = tc::desc_adv(ad0, k * (AMN ? 2048 : 32));
              const uint64_t bd = tc::desc_adv(bd0, k * (BMN ? 2048 : 32));
              const uint32_t acc = (kb != kb0 || k != 0) ? 1u : 0u;
              if (CG == 2)
                mma_bf16_pair(dacc, ad, bd, idesc, acc);
              else
                tc::mma_bf16(dacc, ad, bd, idesc, acc);
            }
            if (CG == 2)
              mma_commit_pair(&empty[s]);
            else
              tc::mma_commit(&empty[s]);
          }
          __syncwarp();
        }
        if (lane == 0) {
          if (CG == 2)
            mma_commit_pair(&tfull[as]);
          else
            tc::mma_commit(&tfull[as]);
          WG_STAMP(it, 1);
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 2;
    const int q = warp & 3;            // TMEM lane quarter this warp may access
    const int chalf = ew >> 2;         // column slice of the 256-wide tile
    constexpr int CW = OUTF32 ? 16 : 32;   // columns per 64-byte chunk
    constexpr int NCH = kSliceCols / CW;
    unsigned char* stg = sStg + ew * kNBuf * kStg;
    uint64_t* xb = xbar + 2 * ew;
    const bool aux = kAux || p.beta;
    const uint32_t tempty_c = CG == 2 ? mapa(&tempty[0], 0) : 0;   // leader's barriers
    // chunk c of unit u: output coordinates
    auto chunk_coords = [&](int u, int c, int& row0, int& col) {
      int mb, nb, sp;
      decode(p, u, mb, nb, sp);
      row0 = mb * kBM * CG + rank * kBM + q * 32;
      col = nb * kBN + chalf * kSliceCols + c * CW;
    };
    auto issue_aux = [&](int u, int c, int buf) {
      int row0, col;
      chunk_coords(u, c, row0, col);
      mbar_arrive_expect_tx(&xb[buf], kStg);
      tc::tma_load_2d(stg + buf * kStg, &mapX, &xb[buf], col, row0);
    };
    uint32_t cidx = 0;   // chunks processed by this warp (buffer parity, aux barrier phase)
    if (aux && lane == 0 && cid < p.units) issue_aux(cid, 0, 0);
    int it = 0;
    for (int u = cid; u < p.units; u += ncl, ++it) {
      int mb, nb, sp;
      decode(p, u, mb, nb, sp);
      const int as = it & 1;
      mbar_wait_sleep(&tfull[as], (it >> 1) & 1, 20000u);
      tc::fence_after_sync();
      if (ew == 0 && lane == 0) WG_STAMP(it, 2);
      const int row0 = mb * kBM * CG + rank * kBM + q * 32;
      const int row = row0 + lane;
      const int out_row0 = row0 + sp * p.M;   // split-K partial slab (EPI_STORE, fp32)
      const int prow = (mb * CG + (int)rank) * 4 + q;   // column-partial row (EPI_BAD_BWD)
#pragma unroll 1
      for (int c = 0; c < NCH; ++c, ++cidx) {
        const int col = nb * kBN + chalf * kSliceCols + c * CW;
        // staging buffer of this chunk (EPI_BAD_FWD: both, h and A1)
        const int buf = cidx & 1;
        unsigned char* sb = stg + buf * kStg;
        unsigned char* sb2 = stg + (buf ^ 1) * kStg;
        // BAD epilogues with stored keep bytes: this lane's word (4 chunks of its row), loaded
        // before the accumulator so its latency hides behind the TMEM load
        uint32_t kw_pre = 0;
        if ((EPI == EPI_BAD_FWD || EPI == EPI_BAD_BWD) && p.kb_in != nullptr && row < p.M &&
            col < p.N) {
          const int64_t ci0 = (int64_t)row * (p.N >> 3) + (col >> 3);
          if ((p.N & 31) == 0) {
            kw_pre = __ldg(reinterpret_cast<const uint32_t*>(p.kb_in + ci0));
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (col + 8 * j < p.N) kw_pre |= (uint32_t)__ldg(p.kb_in + ci0 + j) << (8 * j);
          }
        }
        float v[CW];
        const uint32_t taddr =
            tmem + ((uint32_t)(q * 32) << 16) + as * kBN + chalf * kSliceCols + c * CW;
        if (CW == 32)
          tc::tmem_ld32(taddr, v);
        else
          tc::tmem_ld16(taddr, v);
        if (c == NCH - 1) {   // accumulator drained: the MMA warp may reuse it
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) {
            if (CG == 2)
              mbar_arrive_cluster(tempty_c + as * 8);
            else
              mbar_arrive(&tempty[as]);
          }
        }
        // results are formed in registers first, so the stores issued from the staging
        // buffers by earlier chunks drain while this chunk computes
        uint4 o0[4], o1[4];
        if (aux) mbar_wait(&xb[cidx & 1], (cidx >> 1) & 1);
        if (EPI == EPI_STORE) {
          if (p.bias != nullptr) {
#pragma unroll
            for (int j = 0; j < CW; j += 8) {
              float b[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
              if (col + j < p.N) load_f32x8(p.bias + col + j, b);
#pragma unroll
              for (int i = 0; i < 8; ++i) v[j + i] += b[i];
            }
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (OUTF32) {
              o0[j] = make_uint4(__float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]),
                                 __float_as_uint(v[4 * j + 2]), __float_as_uint(v[4 * j + 3]));
            } else {
              if (p.beta) {
                float r[8];
                unpack_bf16x8(*reinterpret_cast<const uint4*>(sb + sw64(lane, j)), r);
#pragma unroll
                for (int i = 0; i < 8; ++i) v[8 * j + i] += r[i];
              }
              o0[j] = pack_bf16x8(v + 8 * j);
            }
          }
        } else if (EPI == EPI_BAD_FWD) {
          // h = acc + b1 (stored, bf16); A1 = keep ? act(h) * s : 0 from the stored h
          PhiloxKey pkh = p.pk;
          pkh.scale *= 0.5f;   // act_f2 returns 2 act(h)
          const int64_t ci0 = (int64_t)row * (p.N >> 3) + (col >> 3);   // first chunk
          uint32_t kw = kw_pre;   // its 4 keep bytes (given, R29; or formed below)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float b[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, hb[8], m[8], a[8];
            if (col + 8 * j < p.N) load_f32x8(p.bias + col + 8 * j, b);
#pragma unroll
            for (int i = 0; i < 8; ++i) hb[i] = v[8 * j + i] + b[i];
            o0[j] = pack_bf16x8(hb);
            unpack_bf16x8(o0[j], hb);
            if (p.kb_in != nullptr)
              mul8_from_byte(kw >> (8 * j), pkh.scale, m);
            else if (p.kb_out != nullptr)
              kw |= keep_byte_mul8((uint64_t)(p.g0 + ci0 + j), pkh, m) << (8 * j);
            else
              keep_mul8((uint64_t)(p.g0 + ci0 + j), pkh, m);
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = act_f2<ACT>(hb[i]) * m[i];
            o1[j] = pack_bf16x8(a);
          }
          if (p.kb_out != nullptr && row < p.M && col < p.N) {
            if ((p.N & 31) == 0) {   // whole, 4-B aligned words
              *reinterpret_cast<uint32_t*>(p.kb_out + ci0) = kw;
            } else {
#pragma unroll
              for (int j = 0; j < 4; ++j)
                if (col + 8 * j < p.N) p.kb_out[ci0 + j] = (uint8_t)(kw >> (8 * j));
            }
          }
        }
        if (EPI != EPI_BAD_BWD) {
          if (!aux) {
            // the stores issued from these buffers two chunks ago must have read them
            if (lane == 0) {
              if (EPI == EPI_BAD_FWD)
                tc::bulk_wait_read<0>();
              else
                tc::bulk_wait_read<1>();
            }
            __syncwarp();
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            *reinterpret_cast<uint4*>(sb + sw64(lane, j)) = o0[j];
            if (EPI == EPI_BAD_FWD) *reinterpret_cast<uint4*>(sb2 + sw64(lane, j)) = o1[j];
          }
        } else {   // EPI_BAD_BWD
          // dh = keep ? acc * s * act'(h) : 0, written over h in the staging buffer
          const int64_t ci0 = (int64_t)row * (p.N >> 3) + (col >> 3);   // first chunk
          const uint32_t kw = kw_pre;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float h8[8], m[8];
            unpack_bf16x8(*reinterpret_cast<const uint4*>(sb + sw64(lane, j)), h8);
            if (p.kb_in != nullptr)
              mul8_from_byte(kw >> (8 * j), p.pk.scale, m);
            else
              keep_mul8((uint64_t)(p.g0 + ci0 + j), p.pk, m);
#pragma unroll
            for (int i = 0; i < 8; ++i) v[8 * j + i] = v[8 * j + i] * m[i] * act_df<ACT>(h8[i]);
            *reinterpret_cast<uint4*>(sb + sw64(lane, j)) = pack_bf16x8(v + 8 * j);
          }
          // column sums over this warp's 32 rows: transpose-reduce, lane l ends with column l
#pragma unroll
          for (int s = 16; s >= 1; s >>= 1) {
            const bool up = (lane & s) != 0;
#pragma unroll
            for (int i = 0; i < s; ++i) {
              const float send = up ? v[i] : v[i + s];
              const float keep = up ? v[i + s] : v[i];
              v[i] = keep + __shfl_xor_sync(0xFFFFFFFFu, send, s);
            }
          }
          if (col + lane < p.N) p.partials[(int64_t)prow * p.N + col + lane] = v[0];
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tc::tma_store_2d(&mapC, sb, col, out_row0);
          if (EPI == EPI_BAD_FWD) tc::tma_store_2d(&mapC2, sb2, col, row0);
          tc::bulk_commit();
          if (aux) {
            // prefetch the next chunk's auxiliary tile into the other buffer once the store
            // issued from it (previous chunk) has read it
            int nu = u, nc = c + 1;
            if (nc == NCH) {
              nc = 0;
              nu = u + ncl;
            }
            if (nu < p.units) {
              tc::bulk_wait_read<1>();
              issue_aux(nu, nc, (cidx + 1) & 1);
            }
          }
        }
        __syncwarp();
      }
      if (ew == 0 && lane == 0) WG_STAMP(it, 3);
      (void)row;
    }
    if (lane == 0) tc::bulk_wait<0>();
    __syncwarp();
  }
  tc::fence_before_sync();
  if (CG == 2) {
    cluster_sync();   // both CTAs done with the pair's TMEM and barriers
    if (warp == 1)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem)
                   : "memory");
  } else {
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tmem, 512);
  }
}

// split-K partial slabs [splits][M][N] fp32 -> C, summed in split order (deterministic)
__global__ void splitk_reduce_kernel(const float4* __restrict__ ws, float4* __restrict__ C,
                                     int64_t n4, int splits) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 a = ws[i];
    for (int s = 1; s < splits; ++s) {
      const float4 b = ws[(int64_t)s * n4 + i];
      a.x += b.x;
      a.y += b.y;
      a.z += b.z;
      a.w += b.w;
    }
    C[i] = a;
  }
}

}  // namespace wg

// ------------------------------------------------------------------ host side
namespace {
bool map2d(CUtensorMap* m, const void* ptr, bool f32, uint64_t inner, uint64_t outer, int64_t ld,
           uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle sw) {
  const int es = f32 ? 4 : 2;
  if (((uintptr_t)ptr & 15u) || ((ld * es) & 15) || inner == 0 || outer == 0) return false;
  cuuint64_t gdim[2] = {inner, outer};
  cuuint64_t gstr[1] = {(cuuint64_t)ld * es};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es1[2] = {1, 1};
  return tmap_encode_tiled(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                           2, const_cast<void*>(ptr), gdim, gstr, box, es1,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int CG, int AMN, int BMN, int OUTF32, int EPI, int ACT>
cudaError_t launch_t(int grid, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c,
                     const CUtensorMap& c2, const CUtensorMap& x, const wg::Params& p,
                     cudaStream_t st) {
  auto kern = wg::wgemm_kernel<CG, AMN, BMN, OUTF32, EPI, ACT>;
  constexpr size_t smem = wg::Cfg<CG, EPI>::kSmem;
  static bool attr = false;   // per instantiation
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (CG == 1) return launch_k(PDL_WGEMM, kern, grid, wg::kThreads, smem, st, a, b, c, c2, x, p);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(wg::kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled(PDL_WGEMM) ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, a, b, c, c2, x, p);
}
}  // namespace

bool wgemm_supported(const WgemmArgs& g) {
  if (g.M <= 0 || g.N <= 0 || g.K <= 0 || g.N % 8 || g.K % 8 || !g.A || !g.B || !g.C)
    return false;
  switch (g.epi) {
    case EPI_STORE:
      return !(g.beta && g.out_f32);
    case EPI_BAD_FWD:
      return g.bias && g.C2 && !g.out_f32 && !g.beta && !g.a_mn && !g.b_mn;
    case EPI_BAD_BWD:
      return g.aux && g.partials && !g.out_f32 && !g.beta && !g.a_mn && g.b_mn;
    default:
      return false;
  }
}

// CTA pairs (256-row tiles) unless the caller asked for single CTAs or the problem is a
// single 128-row block
static int pick_cg(const WgemmArgs& g) { return g.cg == 1 || g.M <= wg::kBM ? 1 : 2; }

// split count for an fp32 output: minimise (waves x k-blocks per split) + the reduce pass
static int choose_splits(int tiles, int nk, int slots, int64_t MN) {
  int best = 1;
  double best_cost = 1e300;
  for (int s = 1; s <= 8; ++s) {
    const int kbs = (nk + s - 1) / s;
    if (s > 1 && (kbs < 4 || (int64_t)(s - 1) * kbs >= nk)) break;
    const double waves = (double)((tiles * s + slots - 1) / slots);
    // one k-block of one tile ~ 0.3 us of MMA; the reduce reads s+1 slabs of M*N fp32 at
    // ~4 TB/s (mostly L2-resident)
    const double cost = waves * kbs * 0.3 + (s > 1 ? (double)(s + 1) * MN * 4 / 4.0e6 : 0.0);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = s;
    }
  }
  return best;
}

namespace {
struct Plan {
  int cg, tiles_m, tiles_n, nk, splits;
};
Plan plan_of(const WgemmArgs& g, int num_sms) {
  Plan P;
  P.cg = pick_cg(g);
  P.tiles_m = (g.M + wg::kBM * P.cg - 1) / (wg::kBM * P.cg);
  P.tiles_n = (g.N + wg::kBN - 1) / wg::kBN;
  P.nk = (g.K + wg::kBK - 1) / wg::kBK;
  P.splits = 1;
  if (g.epi == EPI_STORE && g.out_f32 && g.ws)
    P.splits = choose_splits(P.tiles_m * P.tiles_n, P.nk, num_sms / P.cg, (int64_t)g.M * g.N);
  // the partial slabs are stacked along M: only whole M tiles keep them apart
  if (P.splits > 1 && (g.M % (wg::kBM * P.cg) ||
                       g.ws_bytes < (size_t)P.splits * g.M * g.N * sizeof(float)))
    P.splits = 1;
  return P;
}
}  // namespace

int wgemm_partial_rows(const WgemmArgs& g) {
  const int cg = pick_cg(g);
  return ((g.M + wg::kBM * cg - 1) / (wg::kBM * cg)) * cg * 4;
}

cudaError_t launch_wgemm(const WgemmArgs& g, int num_sms, cudaStream_t st) {
  if (!wgemm_supported(g)) return cudaErrorInvalidValue;
  const Plan P = plan_of(g, num_sms);
  wg::Params p{};
  p.M = g.M;
  p.N = g.N;
  p.K = g.K;
  p.tiles_m = P.tiles_m;
  p.tiles_n = P.tiles_n;
  p.nk = P.nk;
  p.splits = P.splits;
  p.kb_per_split = (p.nk + p.splits - 1) / p.splits;
  p.units = p.tiles_m * p.tiles_n * p.splits;
  p.beta = g.beta;
  p.bias = g.bias;
  p.pk = g.pk;
  p.g0 = g.g0;
  p.partials = g.partials;
  p.kb_out = g.kb_out;
  p.kb_in = g.kb_in;

  CUtensorMap ma, mb, mc, mc2, mx;
  bool ok = true;
  const auto SW128 = CU_TENSOR_MAP_SWIZZLE_128B, SW64 = CU_TENSOR_MAP_SWIZZLE_64B;
  // A: K-major [M][K] (box 64 x 128) or MN-major [K][M] (box 64 x 64, two per stage);
  // B: this CTA's 256/CG columns the same way
  const uint32_t bcols = wg::kBN / P.cg;
  ok &= g.a_mn ? map2d(&ma, g.A, false, g.M, g.K, g.lda, 64, 64, SW128)
               : map2d(&ma, g.A, false, g.K, g.M, g.lda, 64, wg::kBM, SW128);
  ok &= g.b_mn ? map2d(&mb, g.B, false, g.N, g.K, g.ldb, 64, 64, SW128)
               : map2d(&mb, g.B, false, g.K, g.N, g.ldb, 64, bcols, SW128);
  const bool f32 = g.out_f32 != 0;
  const uint32_t cw = f32 ? 16 : 32;
  if (p.splits > 1)
    ok &= map2d(&mc, g.ws, true, g.N, (uint64_t)g.M * p.splits, g.N, cw, 32, SW64);
  else
    ok &= map2d(&mc, g.C, f32, g.N, g.M, g.ldc, cw, 32, SW64);
  mc2 = mc;
  mx = mc;
  if (g.epi == EPI_BAD_FWD) ok &= map2d(&mc2, g.C2, false, g.N, g.M, g.ldc2, 32, 32, SW64);
  if (g.epi == EPI_BAD_BWD) ok &= map2d(&mx, g.aux, false, g.N, g.M, g.ldaux, 32, 32, SW64);
  if (g.beta) ok &= map2d(&mx, g.C, false, g.N, g.M, g.ldc, 32, 32, SW64);
  if (!ok) return cudaErrorInvalidValue;

  const int slots = num_sms / P.cg;
  const int grid = (p.units < slots ? p.units : slots) * P.cg;
  cudaError_t e = cudaErrorInvalidValue;
#define WG_LAUNCH1(CG, AM, BM, OF, EP, AC) \
  e = launch_t<CG, AM, BM, OF, EP, AC>(grid, ma, mb, mc, mc2, mx, p, st)
#define WG_LAUNCH(AM, BM, OF, EP, AC)            \
  do {                                           \
    if (P.cg == 2) WG_LAUNCH1(2, AM, BM, OF, EP, AC); \
    else WG_LAUNCH1(1, AM, BM, OF, EP, AC);       \
  } while (0)
  if (g.epi == EPI_STORE) {
    if (!g.a_mn && !g.b_mn && !f32) WG_LAUNCH(0, 0, 0, EPI_STORE, 0);
    else if (!g.a_mn && g.b_mn && !f32) WG_LAUNCH(0, 1, 0, EPI_STORE, 0);
    else if (g.a_mn && g.b_mn && f32) WG_LAUNCH(1, 1, 1, EPI_STORE, 0);
    else if (!g.a_mn && !g.b_mn && f32) WG_LAUNCH(0, 0, 1, EPI_STORE, 0);
    else return cudaErrorInvalidValue;
  } else if (g.epi == EPI_BAD_FWD) {
    if (g.a_mn || g.b_mn) return cudaErrorInvalidValue;
    ENC_ACT_DISPATCH(g.act, WG_LAUNCH(0, 0, 0, EPI_BAD_FWD, ACT));
  } else {
    if (g.a_mn || !g.b_mn) return cudaErrorInvalidValue;
    ENC_ACT_DISPATCH(g.act, WG_LAUNCH(0, 1, 0, EPI_BAD_BWD, ACT));
  }
#undef WG_LAUNCH
#undef WG_LAUNCH1
  if (e != cudaSuccess || p.splits == 1) return e;
  const int64_t n4 = (int64_t)g.M * g.N / 4;
  int64_t blocks = (n4 + 255) / 256;
  if (blocks > 8 * num_sms) blocks = 8 * num_sms;
  wg::splitk_reduce_kernel<<<(int)blocks, 256, 0, st>>>((const float4*)g.ws, (float4*)g.C, n4,
                                                        p.splits);
  return cudaGetLastError();
}

int wgemm_launches(const WgemmArgs& g, int num_sms) {
  return plan_of(g, num_sms).splits > 1 ? 2 : 1;
}

#ifdef ENC_WGEMM_TRACE
extern "C" int enc_debug_wgemm_trace(void* host, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(host, wg::g_wg_trace, bytes);
}
extern "C" int enc_debug_wgemm_trace_clear() {
  static unsigned long long zero[148 * 8 * 4];
  return (int)cudaMemcpyToSymbol(wg::g_wg_trace, zero, sizeof(zero));
}
#endif

}  // namespace enc

// Per-(b, h) tcgen05 contractions over the attention-probability tensors (Table A.1
// PAPER.md:553 "Gamma", and its backward dX1/dX2 rows :588-592):
//
//   AV    C[j,:]  = sum_k A[j,k]  V[k,:]        (forward, A = dropout(P))
//   dV    dV[k,:] = sum_j A[j,k]  dC[j,:]
//   dQdK  dQ[j,:] = sum_k dS[j,k] K[k,:]  and  dK[k,:] = sum_j dS[j,k] Q[j,:]   (one pass)
//
// These four contractions read a [J x K] = 512 KB bf16 matrix per (b, h) and write only
// 64 KB, so they are HBM-bound on that read (67 MB at config L).  One CTA owns a whole
// (b, h) pair: it streams the matrix once in 128 x 128 blocks through a TMA ring, and every
// output row tile stays resident in TMEM until the pair is done (J/128 x 64 columns per
// output, <= 512 columns for dQ and dK together).  dQ and dK share each dS block, so dS
// is read once instead of twice.  The same smem block serves as a K-major operand (row
// outputs: C, dQ) and as an MN-major operand (column outputs: dV, dK).
//
// Warp roles (192 threads, one CTA per SM, persistent over (b, h) pairs):
//   warp 0     TMA producer      warp 1  TMEM allocator + MMA issuer
//   warps 2-5  epilogue: TMEM -> bf16 -> 128-B-swizzled staging -> TMA store
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.h"
#include "tc_gemm.cuh"

namespace enc {
namespace {

constexpr int kXfWarps = 8;   // dropout-on-load: zero the dropped elements of each X block
constexpr int kThreads = 192 + kXfWarps * 32;
constexpr uint32_t kXBytes = 128 * 128 * 2;  // one 128 x 128 block (two 64-column boxes)
constexpr uint32_t kYBytes = 128 * 64 * 2;   // one 128-row x 64 operand block

struct BhParams {
  int H, nt;           // heads, J / 128
  int units;           // B * H
  int row_out, col_out;  // which outputs this launch computes
  int yr_rowdim, yc_rowdim, or_rowdim, oc_rowdim;  // 4-D map dim holding the row index
  // optional column sums of the (bf16-rounded) row / column outputs over their rows:
  // ps_*[(b * 4 + quarter) * ps_ld + h * 64 + c], summed over b and quarter afterwards
  float* ps_r;
  float* ps_c;
  int ps_ld;
  // dropout applied on load (A = keep ? P * s : 0 from the stored P and keep words): the
  // transform warps zero the dropped elements of each X block in shared memory before the
  // MMA, and the epilogue multiplies the fp32 accumulators by out_scale (= s)
  const uint32_t* keep;   // [B*H*J, K/32] ENC_KEEP_BITS words, or null (X used as is)
  float out_scale;
  // keep_gen (A.V only, R28): the words are not read but generated from the Philox stream
  // of the attention dropout site (key pk, chunk g0 of element (0,0,0,0)) by the
  // dropout-on-load warps, applied, and written to `keep` for the backward
  int keep_gen;
  PhiloxKey pk;
  int64_t g0;
  // optional (row output only): the rounding residual lo = bf16(acc - float(bf16(acc))) of
  // every stored element, same layout as the row output (the attention output's low word
  // for the backward's row term, R26)
  __nv_bfloat16* lo_r;
  int64_t ld_lo;
};

// 0xFFFF / 0x0000 per 16-bit half from the sign bits 15 and 31 (prmt sign replication)
__device__ __forceinline__ uint32_t half_mask(uint32_t g) {
  uint32_t m;
  asm("prmt.b32 %0, %1, 0, 0xBB99;" : "=r"(m) : "r"(g));
  return m;
}

__device__ __forceinline__ void coords(int rowdim, int inner, int row, int h, int b, int* c) {
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

template <int STAGES>
__global__ void __launch_bounds__(kThreads, 1) attn_bh_kernel(
    const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapYr,
    const __grid_constant__ CUtensorMap mapYc, const __grid_constant__ CUtensorMap mapOr,
    const __grid_constant__ CUtensorMap mapOc, BhParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = tc::align1024(smem_raw);
  const uint32_t stage_bytes = kXBytes + (p.row_out ? kYBytes : 0) + (p.col_out ? kYBytes : 0);
  unsigned char* stg_all = base + STAGES * stage_bytes;        // 4 warps x 2 x 4 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(stg_all + 4 * 2 * 4096);
  uint64_t* empty = full + STAGES;
  uint64_t* tm_full = empty + STAGES;   // [4]: outer tile o of the streamed output done
  uint64_t* tm_empty = tm_full + 4;
  uint64_t* xf = tm_empty + 1;           // [STAGES]: X block masked (dropout on load)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xf + STAGES);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nt = p.nt;
  const int nblk = nt * nt;
  const uint32_t col_off = p.row_out ? nt * 64 : 0;   // TMEM column of the column outputs
  // Block order: the outer index is the row tile of the output that completes tile by tile
  // (jt for C / dQ, kt when dV is the only output), so its epilogue overlaps the rest of the
  // stream; with both dQ and dK, dK finishes with the last block.
  const bool col_outer = p.col_out && !p.row_out;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&mapX);
    if (p.row_out) tc::prefetch_tmap(&mapYr), tc::prefetch_tmap(&mapOr);
    if (p.col_out) tc::prefetch_tmap(&mapYc), tc::prefetch_tmap(&mapOc);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int o = 0; o < 4; ++o) mbar_init(&tm_full[o], 1);
    mbar_init(tm_empty, 4);
    for (int s = 0; s < STAGES; ++s) mbar_init(&xf[s], kXfWarps);
    fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();   // operands are the stream predecessor's outputs

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int g = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        const int b = u / p.H, h = u - (u / p.H) * p.H;
        for (int blk = 0; blk < nblk; ++blk, ++g) {
          const int o = blk / nt, i = blk - (blk / nt) * nt;
          const int jt = col_outer ? i : o, kt = col_outer ? o : i;
          const int s = g % STAGES;
          mbar_wait(&empty[s], ((g / STAGES) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[s], stage_bytes);
          unsigned char* sx = base + s * stage_bytes;
          // X block rows jt*128.., columns kt*128.. as two 64-column boxes
          tc::tma_load_4d(sx, &mapX, &full[s], kt * 128, jt * 128, h, b);
          tc::tma_load_4d(sx + 16384, &mapX, &full[s], kt * 128 + 64, jt * 128, h, b);
          unsigned char* sy = sx + kXBytes;
          int c[4];
          if (p.row_out) {   // Yr rows kt*128.. (keys)
            coords(p.yr_rowdim, 0, kt * 128, h, b, c);
            tc::tma_load_4d(sy, &mapYr, &full[s], c[0], c[1], c[2], c[3]);
            sy += kYBytes;
          }
          if (p.col_out) {   // Yc rows jt*128.. (queries)
            coords(p.yc_rowdim, 0, jt * 128, h, b, c);
            tc::tma_load_4d(sy, &mapYc, &full[s], c[0], c[1], c[2], c[3]);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_r = tc::instr_desc_bf16_f32(128, 64, false, true);
    constexpr uint32_t idesc_c = tc::instr_desc_bf16_f32(128, 64, true, true);
    int g = 0, it = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++it) {
      mbar_wait(tm_empty, (it & 1) ^ 1);   // epilogue released the accumulators
      tc::fence_after_sync();
      for (int blk = 0; blk < nblk; ++blk, ++g) {
        const int o = blk / nt, i = blk - (blk / nt) * nt;
        const int jt = col_outer ? i : o, kt = col_outer ? o : i;
        const int s = g % STAGES;
        mbar_wait(p.keep ? &xf[s] : &full[s], (g / STAGES) & 1);
        tc::fence_after_sync();
        if (lane == 0) {
          const uint32_t x0 = smem_u32(base + s * stage_bytes);
          uint32_t y0 = x0 + kXBytes;
          if (p.row_out) {
            // out_r[jt] += X(jt,kt) Yr(kt): X K-major (rows j), Yr MN-major (rows k)
            const uint64_t xd = tc::smem_desc(x0, 16, 1024), yd = tc::smem_desc(y0, 8192, 1024);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
              tc::mma_bf16(tmem + jt * 64, tc::desc_adv(xd, (ks >> 2) * 16384 + (ks & 3) * 32),
                           tc::desc_adv(yd, ks * 2048), idesc_r, (kt | ks) != 0);
            y0 += kYBytes;
          }
          if (p.col_out) {
            // out_c[kt] += X(jt,kt)^T Yc(jt): X MN-major (M = k), Yc MN-major (rows j)
            const uint64_t xd = tc::smem_desc(x0, 16384, 1024), yd = tc::smem_desc(y0, 8192, 1024);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
              tc::mma_bf16(tmem + col_off + kt * 64, tc::desc_adv(xd, ks * 2048),
                           tc::desc_adv(yd, ks * 2048), idesc_c, (jt | ks) != 0);
          }
          tc::mma_commit(&empty[s]);
          if (i == nt - 1) tc::mma_commit(&tm_full[o]);   // outer tile o complete
        }
        __syncwarp();
      }
    }
  } else if (warp >= 6) {
    // ------------------------------------------------------------ dropout on load
    // thread t of the 256 masks row t / 2, 64-column box t % 2 (8 chunks of 8 elements)
    if (p.keep != nullptr) {
      const int tt = (warp - 6) * 32 + lane;
      const int row = tt >> 1, bx = tt & 1;
      // keep words of this thread's row and 64 columns for block (u, blk)
      auto kw_ptr = [&](int u, int blk) {
        const int o = blk / nt, i = blk - (blk / nt) * nt;
        const int jt = col_outer ? i : o, kt = col_outer ? o : i;
        return reinterpret_cast<const uint2*>(
            p.keep + ((int64_t)u * (nt * 128) + jt * 128 + row) * (nt * 4) + kt * 4 + bx * 2);
      };
      const bool hiT = p.pk.T >= 0x8000u;
      const uint32_t C2 = (hiT ? 0x10000u - p.pk.T : 0x8000u - p.pk.T) * 0x10001u;
      const uint32_t Xm = hiT ? 0u : 0xFFFFFFFFu;
      // one block: its keep words kw (read or generated), the dropped elements of its X
      // tile zeroed in shared memory, then handed to the MMA issuer
      auto process = [&](int u, int blk, int g, uint2 kwv) {
        const int s = g % STAGES;
        uint32_t kw[2] = {kwv.x, kwv.y};
        if (p.keep_gen) {
          // this row's 64 columns of block blk: 8 Philox chunks, computed before the wait
          // for the block's data (they do not depend on it); written for the backward
          const int o = blk / nt, i = blk - (blk / nt) * nt;
          const int jt = col_outer ? i : o, kt = col_outer ? o : i;
          const int64_t grow = p.g0 + ((int64_t)u * (nt * 128) + jt * 128 + row) * (nt * 16) +
                               kt * 16 + bx * 8;
          if (p.pk.T == 0) {
            kw[0] = kw[1] = 0xFFFFFFFFu;
          } else {
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              uint32_t f = 0;
#pragma unroll
              for (int j = 0; j < 4; ++j)
                f |= keep_flags((uint64_t)(grow + 4 * c + j), p.pk, C2, Xm, 4 * j);
              kw[c] = f;
            }
          }
          __stcs(const_cast<uint2*>(kw_ptr(u, blk)), make_uint2(kw[0], kw[1]));
        }
        mbar_wait(&full[s], (g / STAGES) & 1);
        unsigned char* sx = base + s * stage_bytes + bx * 16384;
        // only 8-element chunks with a dropped element are rewritten (at p = 0.1, 43 % of
        // the chunks keep all 8)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint32_t f = kw[c >> 2];
          const int j = c & 3;
          const uint32_t all = 0xF000F000u >> (4 * j);
          if ((f & all) != all) {
            uint4* loc = reinterpret_cast<uint4*>(sx + tc::sw128(row, c));
            uint4 x = *loc;
            x.x &= half_mask(f << (4 * j + 0));
            x.y &= half_mask(f << (4 * j + 1));
            x.z &= half_mask(f << (4 * j + 2));
            x.w &= half_mask(f << (4 * j + 3));
            *loc = x;
          }
        }
        fence_proxy_async_smem();   // generic-proxy writes -> visible to the tensor core
        __syncwarp();
        if (lane == 0)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&xf[s]))
                       : "memory");
      };
      // read words: a two-register ring, each word pair loaded two blocks ahead of its use and
      // never moved between registers (the load's latency hides behind a whole block)
      auto load_kw = [&](int u, int blk) {
        return (!p.keep_gen && blk < nblk) ? __ldg(kw_ptr(u, blk)) : make_uint2(0, 0);
      };
      int g = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        uint2 kwa = load_kw(u, 0), kwb = load_kw(u, 1);
        for (int blk = 0; blk < nblk; blk += 2, g += 2) {
          process(u, blk, g, kwa);
          kwa = load_kw(u, blk + 2);
          if (blk + 1 < nblk) {
            process(u, blk + 1, g + 1, kwb);
            kwb = load_kw(u, blk + 3);
          }
        }
        if (nblk & 1) --g;   // the loop counted one block past an odd block count
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;
    unsigned char* stg = stg_all + q * 2 * 4096;
    int it = 0, n = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++it) {
      const int b = u / p.H, h = u - (u / p.H) * p.H;
      const int ngroups = (p.row_out ? nt : 0) + (p.col_out ? nt : 0);
      float sr0 = 0.f, sr1 = 0.f, sc0 = 0.f, sc1 = 0.f;   // column sums (row / col output)
#pragma unroll 1
      for (int gi = 0; gi < ngroups; ++gi, ++n) {
        const bool is_r = p.row_out && gi < nt;
        const int t = p.row_out && !is_r ? gi - nt : gi;   // row tile of this output group
        // groups 0..nt-1 are the streamed output's tiles (outer order); the remaining
        // (dK with dQ) need the last block
        mbar_wait(&tm_full[gi < nt ? gi : nt - 1], it & 1);
        tc::fence_after_sync();
        unsigned char* buf = stg + (n & 1) * 4096;
        if (lane == 0) tc::bulk_wait_read<1>();
        __syncwarp();
        float v[64];
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + gi * 64;
        tc::tmem_ld32(taddr, v);
        tc::tmem_ld32(taddr + 32, v + 32);
        if (p.out_scale != 1.f) {
#pragma unroll
          for (int i = 0; i < 64; ++i) v[i] *= p.out_scale;
        }
        if (gi == ngroups - 1) {   // accumulators free for the next (b, h)
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(tm_empty))
                         : "memory");
        }
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          uint4 w;
          w.x = Chunk<__nv_bfloat16>::pack2(v[8 * ch + 0], v[8 * ch + 1]);
          w.y = Chunk<__nv_bfloat16>::pack2(v[8 * ch + 2], v[8 * ch + 3]);
          w.z = Chunk<__nv_bfloat16>::pack2(v[8 * ch + 4], v[8 * ch + 5]);
          w.w = Chunk<__nv_bfloat16>::pack2(v[8 * ch + 6], v[8 * ch + 7]);
          *reinterpret_cast<uint4*>(buf + tc::sw128(lane, ch)) = w;
        }
        if (is_r && p.lo_r != nullptr) {
          // lane = row; its 64 columns are 128 contiguous bytes of the [B,J,H,P] rows
          __nv_bfloat16* lo = p.lo_r + ((int64_t)b * (nt * 128) + t * 128 + q * 32 + lane) *
                                           p.ld_lo + h * 64;
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) {
            float r8[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const float hi = __bfloat162float(__float2bfloat16_rn(v[8 * ch + u]));
              r8[u] = v[8 * ch + u] - hi;
            }
            uint4 w;
            w.x = Chunk<__nv_bfloat16>::pack2(r8[0], r8[1]);
            w.y = Chunk<__nv_bfloat16>::pack2(r8[2], r8[3]);
            w.z = Chunk<__nv_bfloat16>::pack2(r8[4], r8[5]);
            w.w = Chunk<__nv_bfloat16>::pack2(r8[6], r8[7]);
            *reinterpret_cast<uint4*>(lo + ch * 8) = w;
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          int c[4];
          coords(is_r ? p.or_rowdim : p.oc_rowdim, 0, t * 128 + q * 32, h, b, c);
          tc::tma_store_4d(is_r ? &mapOr : &mapOc, buf, c[0], c[1], c[2], c[3]);
          tc::bulk_commit();
        }
        if (is_r ? p.ps_r != nullptr : p.ps_c != nullptr) {
          // column sums of the values as stored (the bf16 staging tile), over this warp's 32
          // rows: lane l reads the bf16 pair of columns (2l, 2l+1) of every row
          float a0 = 0.f, a1 = 0.f;
#pragma unroll 8
          for (int rr = 0; rr < 32; ++rr) {
            const uint32_t w = *reinterpret_cast<const uint32_t*>(
                buf + tc::sw128(rr, lane >> 2) + (lane & 3) * 4);
            a0 += __uint_as_float(w << 16);
            a1 += __uint_as_float(w & 0xFFFF0000u);
          }
          if (is_r) {
            sr0 += a0;
            sr1 += a1;
          } else {
            sc0 += a0;
            sc1 += a1;
          }
        }
      }
      const int64_t pso = (int64_t)(b * 4 + q) * p.ps_ld + h * 64 + 2 * lane;
      if (p.ps_r != nullptr && p.row_out)
        *reinterpret_cast<float2*>(p.ps_r + pso) = make_float2(sr0, sr1);
      if (p.ps_c != nullptr && p.col_out)
        *reinterpret_cast<float2*>(p.ps_c + pso) = make_float2(sc0, sc1);
    }
    if (lane == 0) tc::bulk_wait<0>();
    __syncwarp();
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

bool make_map(CUtensorMap* m, const void* ptr, const uint64_t d[4], const uint64_t s[3],
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

// logical [B*H][rows][cols]; head-major [B][H][rows][cols] (rowdim 1) or token-major
// [B][rows][H][cols] (rowdim 2); box {64 cols, box_rows rows}
bool map_op(CUtensorMap* m, const void* ptr, bool token_major, int B, int H, int rows, int cols,
            int box_rows, int* rowdim) {
  uint64_t d[4], s[3];
  uint32_t box[4];
  if (!token_major) {
    d[0] = cols; d[1] = rows; d[2] = H; d[3] = B;
    s[0] = cols; s[1] = (uint64_t)rows * cols; s[2] = (uint64_t)H * rows * cols;
    box[0] = 64; box[1] = box_rows; box[2] = 1; box[3] = 1;
    *rowdim = 1;
  } else {
    d[0] = cols; d[1] = H; d[2] = rows; d[3] = B;
    s[0] = cols; s[1] = (uint64_t)H * cols; s[2] = (uint64_t)rows * H * cols;
    box[0] = 64; box[1] = 1; box[2] = box_rows; box[3] = 1;
    *rowdim = 2;
  }
  return make_map(m, ptr, d, s, box);
}

int sm_count() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

template <int STAGES>
cudaError_t launch_bh(const CUtensorMap* m, const BhParams& p, cudaStream_t st) {
  const uint32_t stage_bytes = kXBytes + (p.row_out ? kYBytes : 0) + (p.col_out ? kYBytes : 0);
  const size_t smem = 1024 + STAGES * stage_bytes + 4 * 2 * 4096 + (3 * STAGES + 5) * 8 + 16;
  cudaFuncSetAttribute(attn_bh_kernel<STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  const int grid = p.units < sm_count() ? p.units : sm_count();
  launch_k(PDL_ATTN_BH, attn_bh_kernel<STAGES>, grid, kThreads, smem, st, m[0], m[1], m[2], m[3], m[4], p);
  return cudaGetLastError();
}

}  // namespace

// J = K keys, a multiple of 128 up to 512 (every output row tile of a (b, h) in TMEM)
bool attn_bh_supported(int J, int P) { return P == 64 && J % 128 == 0 && J >= 128 && J <= 512; }

// C = A V (AV), dV = A^T dC (DV), dQ = dS K and dK = dS^T Q (DQ / DK, or both from one
// read of dS).  P-wide operands take row strides (kernels.h, map_pop).
static cudaError_t bh_launch(int B, int H, int J, int P, const void* X, const void* Yr,
                             int64_t ldyr, const void* Yc, int64_t ldyc, void* Or, int64_t ldor,
                             void* Oc, int64_t ldoc, float* ps_r, float* ps_c, int ps_ld,
                             const uint32_t* keep, float out_scale, cudaStream_t st,
                             void* lo_r = nullptr, const PhiloxKey* gen_pk = nullptr,
                             int64_t gen_g0 = 0) {
  if (!attn_bh_supported(J, P)) return cudaErrorInvalidValue;
  if (lo_r && (((uintptr_t)lo_r & 15u) || ldor % 8)) return cudaErrorInvalidValue;
  BhParams p{};
  p.lo_r = (__nv_bfloat16*)lo_r;
  p.ld_lo = ldor;
  p.H = H;
  p.nt = J / 128;
  p.units = B * H;
  p.row_out = Or != nullptr;
  p.col_out = Oc != nullptr;
  p.yr_rowdim = p.yc_rowdim = p.or_rowdim = p.oc_rowdim = 2;   // map_pop: (p, h, row, b)
  p.ps_r = ps_r;
  p.ps_c = ps_c;
  p.ps_ld = ps_ld;
  p.keep = keep;
  p.out_scale = out_scale;
  if (gen_pk != nullptr) {
    p.keep_gen = 1;
    p.pk = *gen_pk;
    p.g0 = gen_g0;
  }
  CUtensorMap m[5];
  int rd;
  bool ok = map_op(&m[0], X, false, B, H, J, J, 128, &rd);
  m[1] = m[0];
  m[2] = m[0];
  m[3] = m[0];
  m[4] = m[0];
  if (p.row_out) {
    ok &= map_pop(&m[1], Yr, B, H, J, P, ldyr, 128);
    ok &= map_pop(&m[3], Or, B, H, J, P, ldor, 32);
  }
  if (p.col_out) {
    ok &= map_pop(&m[2], Yc, B, H, J, P, ldyc, 128);
    ok &= map_pop(&m[4], Oc, B, H, J, P, ldoc, 32);
  }
  if (!ok) return cudaErrorInvalidValue;
  if (p.units == 0) return cudaSuccess;
  if (p.row_out && p.col_out) return launch_bh<3>(m, p, st);
  return launch_bh<4>(m, p, st);
}

cudaError_t launch_attn_av_bh(int B, int H, int J, int P, const void* A, const void* V,
                              int64_t ldv, void* C, int64_t ldc, const uint32_t* keep,
                              float scale, cudaStream_t st, void* C_lo, const PhiloxKey* gen_pk,
                              int64_t batch_offset) {
  return bh_launch(B, H, J, P, A, V, ldv, nullptr, 0, C, ldc, nullptr, 0, nullptr, nullptr, 0,
                   keep, keep ? scale : 1.f, st, C_lo, gen_pk,
                   batch_offset * (int64_t)H * J * (J / 8));
}

cudaError_t launch_attn_dv_bh(int B, int H, int J, int P, const void* A, const void* dC,
                              int64_t lddc, void* dV, int64_t lddv, float* ps_dv, int ps_ld,
                              const uint32_t* keep, float scale, cudaStream_t st) {
  return bh_launch(B, H, J, P, A, nullptr, 0, dC, lddc, nullptr, 0, dV, lddv, nullptr, ps_dv,
                   ps_ld, keep, keep ? scale : 1.f, st);
}

cudaError_t launch_attn_dqdk_bh(int B, int H, int J, int P, const void* dS, const void* Kt,
                                int64_t ldk, const void* Q, int64_t ldq, void* dQ, int64_t lddq,
                                void* dK, int64_t lddk, float* ps_dq, float* ps_dk, int ps_ld,
                                cudaStream_t st) {
  return bh_launch(B, H, J, P, dS, Kt, ldk, Q, ldq, dQ, lddq, dK, lddk, ps_dq, ps_dk, ps_ld,
                   nullptr, 1.f, st);
}

}  // namespace enc

// Shared device helpers for the fused memory-bound operators (sm_100a).
//
// Data unit: a "chunk" = 8 consecutive elements of a row.  bf16: one 16-byte vector
// (LDG.128/STG.128); fp32: two 16-byte vectors.  Every row length (I, U, K, P) is a
// multiple of 8, so chunks never straddle rows and one Philox4x32-10 call yields the 8
// dropout decisions of a chunk (R5: 16-bit lanes, 8 per call).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace enc {

constexpr int kWarp = 32;

// ---------------------------------------------------------------- chunk load / store
// Raw = the chunk's bytes as loaded (kept packed in registers until used, so all loads of
// a row can be issued before any arithmetic: memory-level parallelism).
template <typename T>
struct Chunk;

template <>
struct Chunk<__nv_bfloat16> {
  using Raw = uint4;
  static constexpr int kBytes = 16;
  static __device__ __forceinline__ Raw ld(const __nv_bfloat16* p) {  // streamed once
    return __ldcs(reinterpret_cast<const uint4*>(p));
  }
  static __device__ __forceinline__ Raw ld_smem(const __nv_bfloat16* p) {
    return *reinterpret_cast<const uint4*>(p);
  }
  static __device__ __forceinline__ void unpack(const Raw& u, float v[8]) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  }
  static __device__ __forceinline__ void load_cs(const __nv_bfloat16* p, float v[8]) {
    unpack(ld(p), v);
  }
  static __device__ __forceinline__ uint32_t pack2(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);  // round to nearest even
    return *reinterpret_cast<uint32_t*>(&h);
  }
  static __device__ __forceinline__ void store(__nv_bfloat16* p, const float v[8]) {
    uint4 u;
    u.x = pack2(v[0], v[1]);
    u.y = pack2(v[2], v[3]);
    u.z = pack2(v[4], v[5]);
    u.w = pack2(v[6], v[7]);
    *reinterpret_cast<uint4*>(p) = u;
  }
};

template <>
struct Chunk<float> {
  struct Raw {
    float4 a, b;
  };
  static constexpr int kBytes = 32;
  static __device__ __forceinline__ Raw ld(const float* p) {
    Raw r;
    r.a = __ldcs(reinterpret_cast<const float4*>(p));
    r.b = __ldcs(reinterpret_cast<const float4*>(p) + 1);
    return r;
  }
  static __device__ __forceinline__ Raw ld_smem(const float* p) {
    Raw r;
    r.a = reinterpret_cast<const float4*>(p)[0];
    r.b = reinterpret_cast<const float4*>(p)[1];
    return r;
  }
  static __device__ __forceinline__ void unpack(const Raw& r, float v[8]) {
    v[0] = r.a.x; v[1] = r.a.y; v[2] = r.a.z; v[3] = r.a.w;
    v[4] = r.b.x; v[5] = r.b.y; v[6] = r.b.z; v[7] = r.b.w;
  }
  static __device__ __forceinline__ void load_cs(const float* p, float v[8]) { unpack(ld(p), v); }
  static __device__ __forceinline__ void store(float* p, const float v[8]) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
};

// fp32 parameter vectors (bias, gamma, beta): 8 floats, read through L1 (reused by rows)
__device__ __forceinline__ void load_f32x8(const float* p, float v[8]) {
  float4 a = __ldg(reinterpret_cast<const float4*>(p));
  float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

// ---------------------------------------------------------------- programmatic dependent launch
// A kernel launched with the programmatic-serialization attribute (launch_k, kernels.h) may
// start while its stream predecessor is still running: everything before pdl_wait() (barrier
// init, parameter loads, descriptor prefetch) overlaps the predecessor's tail; pdl_wait()
// returns once the predecessor has completed and its writes are visible.  Without the
// attribute both are no-ops.  pdl_trigger() lets the successor's CTAs launch early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---------------------------------------------------------------- Philox4x32-10
// Salmon et al. SC'11 (Random123); same ctr/key/word layout as cuRAND's
// curand_init(seed, subseq, 4*g) + curand4() (R5).  The ten round keys and the
// counter half that is the same for every call of a site (ctr.zw = subsequence) are
// folded on the host, so a call costs 19 IMAD.WIDE + 20 LOP3 (keys read from the
// kernel-parameter constant bank).
struct PhiloxKey {
  uint32_t rk0[10], rk1[10];  // round keys: seed lo/hi + r * Weyl constants
  uint32_t a0;                // round 0: umulhi(M1, subseq lo) ^ rk0[0]
  uint32_t l1;                // round 0: M1 * subseq lo
  uint32_t b0;                // round 0: subseq hi ^ rk1[0]
  uint32_t T;                 // keep iff 16-bit lane >= T
  float scale;                // 65536 / (65536 - T), correctly rounded
};

__device__ __forceinline__ uint4 philox4x32_10(uint64_t g, const PhiloxKey& pk) {
  const uint32_t g0 = (uint32_t)g, g1 = (uint32_t)(g >> 32);
  // round 0 with ctr = (g0, g1, s0, s1)
  // one IMAD.WIDE.U32 per 32x32->64 product (hi and lo together)
  uint4 c;
  {
    const uint64_t p0 = (uint64_t)0xD2511F53u * g0;
    c = make_uint4(pk.a0 ^ g1, pk.l1, (uint32_t)(p0 >> 32) ^ pk.b0, (uint32_t)p0);
  }
#pragma unroll
  for (int r = 1; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c.x;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c.z;
    c = make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ pk.rk0[r], (uint32_t)p1,
                   (uint32_t)(p0 >> 32) ^ c.w ^ pk.rk1[r], (uint32_t)p0);
  }
  return c;
}

// 8 keep bits (bit i = lane i) of chunk g (= logical index >> 3).  Test hook only; the
// kernels use keep_mul8, which avoids materialising the bits.
__device__ __forceinline__ uint32_t keep_bits8(uint64_t g, const PhiloxKey& pk) {
  if (pk.T == 0) return 0xFFu;
  const uint4 w = philox4x32_10(g, pk);
  const uint32_t T = pk.T;
  const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
  uint32_t b = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    b |= ((wv[i] & 0xFFFFu) >= T) << (2 * i);
    b |= ((wv[i] >> 16) >= T) << (2 * i + 1);
  }
  return b;
}

// m[j] = keep_j ? scale : 0 for the 8 elements of chunk g.  Lane 2i is the low half of
// word i, lane 2i+1 the high half.  r_hi >= T  <=>  w >= T<<16 and r_lo >= T  <=>
// (w << 16) >= T<<16, so each decision is one compare (+ one shift for low halves).
__device__ __forceinline__ void keep_mul8(uint64_t g, const PhiloxKey& pk, float m[8]) {
  if (pk.T == 0) {   // everything kept; pk.scale is 1 for such a key (callers may rescale it)
#pragma unroll
    for (int j = 0; j < 8; ++j) m[j] = pk.scale;
    return;
  }
  const uint4 w = philox4x32_10(g, pk);
  const uint32_t T16 = pk.T << 16;
  const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    m[2 * i] = (wv[i] << 16) >= T16 ? pk.scale : 0.f;
    m[2 * i + 1] = wv[i] >= T16 ? pk.scale : 0.f;
  }
}

// Keep bits of the 8 elements of Philox chunk g (R5: element 2i <-> low 16-bit
// lane of word i, 2i+1 <-> high lane; keep iff lane >= T), as a SWAR compare: with
// C = per-lane (0x8000 - T) for T < 0x8000, x >= T  <=>  x >= 0x8000 or (x & 0x7FFF) + C has
// bit 15 set (no carry leaves a lane), so bit 15 / 31 of ((w & 0x7FFF7FFF) + C) | w is
// the keep bit of the low / high lane.  T >= 0x8000 (p >= 1/2): C = 0x10000 - T and AND.
// The four words' flags are packed as: element u of the chunk -> bit (u odd ? 31 : 15)
// - u/2, then shifted right by `sh`.
// X = all ones for T < 0x8000 (OR), 0 for T >= 0x8000 (AND): (t & w) | ((t | w) & X) is
// one LOP3; the flag bits are then masked as they are merged.
__device__ __forceinline__ uint32_t keep_flags(uint64_t g, const PhiloxKey& pk, uint32_t C2,
                                               uint32_t X, int sh) {
  const uint4 w = philox4x32_10(g, pk);
  const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
  uint32_t f = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t t = (wv[i] & 0x7FFF7FFFu) + C2;
    const uint32_t gi = (t & wv[i]) | ((t | wv[i]) & X);
    f |= (gi >> (i + sh)) & (0x80008000u >> (i + sh));
  }
  return f;
}
// Keep bytes (R27): the 8 keep flags of chunk g as one byte, bit u = element u of
// the chunk, stored by a forward site so its backward reads 1 byte per 8 elements instead
// of re-running Philox.  keep_byte_mul8 also returns the multipliers of keep_mul8.
__device__ __forceinline__ uint32_t keep_byte_mul8(uint64_t g, const PhiloxKey& pk, float m[8]) {
  if (pk.T == 0) {
#pragma unroll
    for (int j = 0; j < 8; ++j) m[j] = pk.scale;
    return 0xFFu;
  }
  const uint4 w = philox4x32_10(g, pk);
  const uint32_t T16 = pk.T << 16;
  const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
  uint32_t b = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool lo = (wv[i] << 16) >= T16, hi = wv[i] >= T16;
    m[2 * i] = lo ? pk.scale : 0.f;
    m[2 * i + 1] = hi ? pk.scale : 0.f;
    b |= (lo ? 1u : 0u) << (2 * i);
    b |= (hi ? 1u : 0u) << (2 * i + 1);
  }
  return b;
}
__device__ __forceinline__ void mul8_from_byte(uint32_t b, float scale, float m[8]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) m[j] = ((b >> j) & 1u) ? scale : 0.f;
}
// multipliers of chunk ci (index within the site, Philox chunk g0 + ci): read from the
// site's stored keep bytes (kb_in), else from Philox -- and then stored to kb_out if given
__device__ __forceinline__ void keep_mul8_io(int64_t g0, int64_t ci, const PhiloxKey& pk,
                                             uint8_t* kb_out, const uint8_t* kb_in, float m[8]) {
  if (kb_in != nullptr) {
    mul8_from_byte(__ldg(kb_in + ci), pk.scale, m);
  } else if (kb_out != nullptr) {
    kb_out[ci] = (uint8_t)keep_byte_mul8((uint64_t)(g0 + ci), pk, m);
  } else {
    keep_mul8((uint64_t)(g0 + ci), pk, m);
  }
}

// v[j] = keep_j ? v[j] * scale : 0
__device__ __forceinline__ void dropout8(float v[8], uint64_t g, const PhiloxKey& pk) {
  if (pk.T == 0) return;
  float m[8];
  keep_mul8(g, pk, m);
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] *= m[j];
}

// ---------------------------------------------------------------- thread-local reductions
// pairwise trees over N (power of 2) register values: log2(N) dependent steps instead of N
template <int N>
__device__ __forceinline__ float tree_sum(const float* v) {
  if constexpr (N == 1) return v[0];
  else return tree_sum<N / 2>(v) + tree_sum<N / 2>(v + N / 2);
}
template <int N>
__device__ __forceinline__ float tree_max(const float* v) {
  if constexpr (N == 1) return v[0];
  else return fmaxf(tree_max<N / 2>(v), tree_max<N / 2>(v + N / 2));
}

// ---------------------------------------------------------------- warp reductions
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
  return v;
}

}  // namespace enc

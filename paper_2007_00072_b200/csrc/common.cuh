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
template <typename T>
struct Chunk;

template <>
struct Chunk<__nv_bfloat16> {
  static __device__ __forceinline__ void load(const __nv_bfloat16* p, float v[8]) {
    uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  }
  // streaming load for data read exactly once
  static __device__ __forceinline__ void load_cs(const __nv_bfloat16* p, float v[8]) {
    uint4 u = __ldcs(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
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
  static __device__ __forceinline__ void store_cs(__nv_bfloat16* p, const float v[8]) {
    uint4 u;
    u.x = pack2(v[0], v[1]);
    u.y = pack2(v[2], v[3]);
    u.z = pack2(v[4], v[5]);
    u.w = pack2(v[6], v[7]);
    __stcs(reinterpret_cast<uint4*>(p), u);
  }
};

template <>
struct Chunk<float> {
  static __device__ __forceinline__ void load(const float* p, float v[8]) {
    float4 a = __ldg(reinterpret_cast<const float4*>(p));
    float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
  static __device__ __forceinline__ void load_cs(const float* p, float v[8]) {
    float4 a = __ldcs(reinterpret_cast<const float4*>(p));
    float4 b = __ldcs(reinterpret_cast<const float4*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
  static __device__ __forceinline__ void store(float* p, const float v[8]) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
  static __device__ __forceinline__ void store_cs(float* p, const float v[8]) {
    __stcs(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3]));
    __stcs(reinterpret_cast<float4*>(p) + 1, make_float4(v[4], v[5], v[6], v[7]));
  }
};

// fp32 parameter vectors (bias, gamma, beta): 8 floats, read through L1 (reused by rows)
__device__ __forceinline__ void load_f32x8(const float* p, float v[8]) {
  float4 a = __ldg(reinterpret_cast<const float4*>(p));
  float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

// ---------------------------------------------------------------- Philox4x32-10
// Salmon et al. SC'11 (Random123); same ctr/key/word layout as cuRAND's
// curand_init(seed, subseq, 4*g) + curand4() (R5).
struct PhiloxKey {
  uint32_t k0, k1;  // seed lo, hi
  uint32_t s0, s1;  // subsequence lo, hi
  uint32_t T;       // keep iff 16-bit lane >= T
  float scale;      // 65536 / (65536 - T), correctly rounded
};

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
  }
  return c;
}

// 8 keep bits (bit i = lane i) of chunk g (= logical index >> 3).
__device__ __forceinline__ uint32_t keep_bits8(uint64_t g, const PhiloxKey& pk) {
  if (pk.T == 0) return 0xFFu;
  const uint4 w = philox4x32_10(make_uint4((uint32_t)g, (uint32_t)(g >> 32), pk.s0, pk.s1),
                                pk.k0, pk.k1);
  const uint32_t T = pk.T;
  uint32_t b = 0;
  b |= ((w.x & 0xFFFFu) >= T) << 0;
  b |= ((w.x >> 16) >= T) << 1;
  b |= ((w.y & 0xFFFFu) >= T) << 2;
  b |= ((w.y >> 16) >= T) << 3;
  b |= ((w.z & 0xFFFFu) >= T) << 4;
  b |= ((w.z >> 16) >= T) << 5;
  b |= ((w.w & 0xFFFFu) >= T) << 6;
  b |= ((w.w >> 16) >= T) << 7;
  return b;
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

// Per-lane vectors of a factor row for the warp-per-rating kernels.
//
// A K-row is spread over the 32 lanes, EPL = K/32 elements per lane, as NV
// vectors of W = min(EPL, 16 bytes / sizeof(S)) consecutive elements;
// vector v of lane l starts at element (v*32 + l)*W.  Every warp-wide vector
// access is therefore one fully coalesced 32*W*sizeof(S)-byte transaction in
// global memory and bank-conflict free in shared memory, for any storage
// width: K=128 fp32 is one 16-byte vector per lane, K=128 fp16 one 8-byte
// vector, K=32 fp32 one 4-byte element.
//
// Vec<S, W> moves W elements as one vector: ldg/red (global, L2-coherent:
// ld.global.cg / red.global.add.v*), lds/sts (shared or generic).  The fp32
// shared-memory Q slice uses the same element interleave (FVec).
#pragma once

#include "hmf_common.cuh"

namespace hmf {

template <typename S, int W> struct Vec;

template <> struct Vec<float, 4> {
  __device__ static void ldg(const float* p, float* o) {
    const float4 v = __ldcg(reinterpret_cast<const float4*>(p));
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
  }
  __device__ static void lds(const float* p, float* o) {
    const float4 v = *reinterpret_cast<const float4*>(p);
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
  }
  __device__ static void stg(float* p, const float* i) {
    __stcg(reinterpret_cast<float4*>(p), make_float4(i[0], i[1], i[2], i[3]));
  }
  __device__ static void sts(float* p, const float* i) {
    *reinterpret_cast<float4*>(p) = make_float4(i[0], i[1], i[2], i[3]);
  }
  __device__ static void red(float* p, const float* d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(d[0]), "f"(d[1]),
                 "f"(d[2]), "f"(d[3])
                 : "memory");
  }
};

template <> struct Vec<float, 2> {
  __device__ static void ldg(const float* p, float* o) {
    const float2 v = __ldcg(reinterpret_cast<const float2*>(p));
    o[0] = v.x; o[1] = v.y;
  }
  __device__ static void lds(const float* p, float* o) {
    const float2 v = *reinterpret_cast<const float2*>(p);
    o[0] = v.x; o[1] = v.y;
  }
  __device__ static void stg(float* p, const float* i) {
    __stcg(reinterpret_cast<float2*>(p), make_float2(i[0], i[1]));
  }
  __device__ static void sts(float* p, const float* i) {
    *reinterpret_cast<float2*>(p) = make_float2(i[0], i[1]);
  }
  __device__ static void red(float* p, const float* d) {
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(d[0]), "f"(d[1])
                 : "memory");
  }
};

template <> struct Vec<float, 1> {
  __device__ static void ldg(const float* p, float* o) { o[0] = __ldcg(p); }
  __device__ static void lds(const float* p, float* o) { o[0] = *p; }
  __device__ static void stg(float* p, const float* i) { __stcg(p, i[0]); }
  __device__ static void sts(float* p, const float* i) { *p = i[0]; }
  __device__ static void red(float* p, const float* d) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(d[0]) : "memory");
  }
};

// fp16 storage: values travel as packed half2 words, computed in fp32.
__device__ inline uint32_t pack_h2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ inline void unpack_h2(uint32_t w, float* o) {
  const float2 f = __half22float2(*reinterpret_cast<__half2*>(&w));
  o[0] = f.x; o[1] = f.y;
}

template <> struct Vec<__half, 8> {
  __device__ static void from(const uint4& v, float* o) {
    unpack_h2(v.x, o); unpack_h2(v.y, o + 2); unpack_h2(v.z, o + 4); unpack_h2(v.w, o + 6);
  }
  __device__ static uint4 to(const float* i) {
    return make_uint4(pack_h2(i[0], i[1]), pack_h2(i[2], i[3]), pack_h2(i[4], i[5]),
                      pack_h2(i[6], i[7]));
  }
  __device__ static void ldg(const __half* p, float* o) {
    from(__ldcg(reinterpret_cast<const uint4*>(p)), o);
  }
  __device__ static void lds(const __half* p, float* o) {
    from(*reinterpret_cast<const uint4*>(p), o);
  }
  __device__ static void stg(__half* p, const float* i) { __stcg(reinterpret_cast<uint4*>(p), to(i)); }
  __device__ static void sts(__half* p, const float* i) { *reinterpret_cast<uint4*>(p) = to(i); }
  __device__ static void red(__half* p, const float* d) {
    const uint4 v = to(d);
    asm volatile("red.global.add.noftz.v4.f16x2 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
  }
};

template <> struct Vec<__half, 4> {
  __device__ static void from(const uint2& v, float* o) { unpack_h2(v.x, o); unpack_h2(v.y, o + 2); }
  __device__ static uint2 to(const float* i) { return make_uint2(pack_h2(i[0], i[1]), pack_h2(i[2], i[3])); }
  __device__ static void ldg(const __half* p, float* o) {
    from(__ldcg(reinterpret_cast<const uint2*>(p)), o);
  }
  __device__ static void lds(const __half* p, float* o) {
    from(*reinterpret_cast<const uint2*>(p), o);
  }
  __device__ static void stg(__half* p, const float* i) { __stcg(reinterpret_cast<uint2*>(p), to(i)); }
  __device__ static void sts(__half* p, const float* i) { *reinterpret_cast<uint2*>(p) = to(i); }
  __device__ static void red(__half* p, const float* d) {
    const uint2 v = to(d);
    asm volatile("red.global.add.noftz.v2.f16x2 [%0], {%1, %2};" ::"l"(p), "r"(v.x), "r"(v.y)
                 : "memory");
  }
};

template <> struct Vec<__half, 2> {
  __device__ static void ldg(const __half* p, float* o) {
    unpack_h2(__ldcg(reinterpret_cast<const unsigned int*>(p)), o);
  }
  __device__ static void lds(const __half* p, float* o) {
    unpack_h2(*reinterpret_cast<const uint32_t*>(p), o);
  }
  __device__ static void stg(__half* p, const float* i) {
    __stcg(reinterpret_cast<unsigned int*>(p), pack_h2(i[0], i[1]));
  }
  __device__ static void sts(__half* p, const float* i) {
    *reinterpret_cast<uint32_t*>(p) = pack_h2(i[0], i[1]);
  }
  __device__ static void red(__half* p, const float* d) {
    asm volatile("red.global.add.noftz.f16x2 [%0], %1;" ::"l"(p), "r"(pack_h2(d[0], d[1]))
                 : "memory");
  }
};

template <> struct Vec<__half, 1> {
  __device__ static void ldg(const __half* p, float* o) {
    o[0] = __half2float(__ushort_as_half(__ldcg(reinterpret_cast<const unsigned short*>(p))));
  }
  __device__ static void lds(const __half* p, float* o) { o[0] = __half2float(*p); }
  __device__ static void stg(__half* p, const float* i) {
    __stcg(reinterpret_cast<unsigned short*>(p), __half_as_ushort(__float2half_rn(i[0])));
  }
  __device__ static void sts(__half* p, const float* i) { *p = __float2half_rn(i[0]); }
  __device__ static void red(__half* p, const float* d) {
    asm volatile("red.global.add.noftz.f16 [%0], %1;" ::"l"(p),
                 "h"(__half_as_ushort(__float2half_rn(d[0])))
                 : "memory");
  }
};

// fp32 vectors of W floats in shared memory (W = 1, 2, 4, 8)
template <int W> struct FVec {
  __device__ static void lds(const float* p, float* o) {
    if constexpr (W >= 4) {
#pragma unroll
      for (int h = 0; h < W / 4; ++h) Vec<float, 4>::lds(p + 4 * h, o + 4 * h);
    } else {
      Vec<float, W>::lds(p, o);
    }
  }
  __device__ static void sts(float* p, const float* i) {
    if constexpr (W >= 4) {
#pragma unroll
      for (int h = 0; h < W / 4; ++h) Vec<float, 4>::sts(p + 4 * h, i + 4 * h);
    } else {
      Vec<float, W>::sts(p, i);
    }
  }
};

template <int K, typename S> struct RowLay {
  static_assert(K % 32 == 0, "K must be a multiple of 32");
  static constexpr int EPL = K / 32;
  static constexpr int WMAX = 16 / int(sizeof(S));
  static constexpr int W = EPL < WMAX ? EPL : WMAX;
  static constexpr int NV = EPL / W;
  using V = Vec<S, W>;
  __device__ static int off(int v, int lane) { return (v * 32 + lane) * W; }

  __device__ static void ldg(const S* row, int lane, float* o) {
#pragma unroll
    for (int v = 0; v < NV; ++v) V::ldg(row + off(v, lane), o + v * W);
  }
  __device__ static void stg(S* row, int lane, const float* i) {
#pragma unroll
    for (int v = 0; v < NV; ++v) V::stg(row + off(v, lane), i + v * W);
  }
  __device__ static void red(S* row, int lane, const float* d) {
    if constexpr (W == 1 && sizeof(S) == 2) {
      // one half per lane: pair neighbouring lanes into a 4-byte f16x2
      // reduction instead of 2-byte atomics (must be called warp-uniformly)
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const float hi = __shfl_down_sync(0xffffffffu, d[v], 1);
        if ((lane & 1) == 0) {
          const float pair[2] = {d[v], hi};
          Vec<S, 2>::red(row + off(v, lane), pair);
        }
      }
    } else {
#pragma unroll
      for (int v = 0; v < NV; ++v) V::red(row + off(v, lane), d + v * W);
    }
  }
  // storage-typed row in shared memory
  __device__ static void lds(const S* row, int lane, float* o) {
#pragma unroll
    for (int v = 0; v < NV; ++v) V::lds(row + off(v, lane), o + v * W);
  }
  __device__ static void sts(S* row, int lane, const float* i) {
#pragma unroll
    for (int v = 0; v < NV; ++v) V::sts(row + off(v, lane), i + v * W);
  }
  // fp32 row in shared memory, same element interleave
  __device__ static void ldsf(const float* row, int lane, float* o) {
#pragma unroll
    for (int v = 0; v < NV; ++v) FVec<W>::lds(row + off(v, lane), o + v * W);
  }
  __device__ static void stsf(float* row, int lane, const float* i) {
#pragma unroll
    for (int v = 0; v < NV; ++v) FVec<W>::sts(row + off(v, lane), i + v * W);
  }
};

}  // namespace hmf
